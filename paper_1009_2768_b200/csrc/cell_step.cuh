// cell_step.cuh — one TRMC-R collision step of one cell, executed by one CTA.
//
// Rows A3..A8 of the hot path (SURVEY §8a / DESIGN.md §3):
//   A3 moments + majorant
//   A4 split into collision sets, Alg 4.2, IR rounding
//   A5 recursive trees of Alg 4.3/4.4 flattened level-synchronously
//   A6 binary / dummy collisions (eq. Maxwell_coll, n3d: P:381-395)
//   A7 TRMC-RAD keep-and-extend
//   A8 conservative Maxwellian of the truncated set
//
// The same routine runs with its working arrays in shared memory (cells up to
// n_cap particles, the fast path) or in global memory (large cells, or a cell
// whose tree overflowed the shared-memory plan; that CTA writes nothing and
// hands the cell to the global-memory kernel).
#pragma once
#include "device_common.cuh"
#include "../../include/trmcr.h"
#include <cooperative_groups.h>

namespace trmcr {

// Optional per-phase cycle accounting (debug builds: -DTRMCR_PHASE_TIMING).
#ifdef TRMCR_PHASE_TIMING
__device__ unsigned long long g_phase_cycles[16];
#define PHASE_MARK(var) long long var = clock64()
#define PHASE_ADD(k, var)                                                        \
  do {                                                                           \
    if (threadIdx.x == 0) atomicAdd(&g_phase_cycles[k], (unsigned long long)(clock64() - var)); \
    var = clock64();                                                             \
  } while (0)
#define WPHASE_ADD(k, var)                                                       \
  do {                                                                           \
    if ((threadIdx.x & 31) == 0) atomicAdd(&g_phase_cycles[k], (unsigned long long)(clock64() - var)); \
    var = clock64();                                                             \
  } while (0)
#else
#define PHASE_MARK(var)
#define PHASE_ADD(k, var)
#define WPHASE_ADD(k, var)
#endif

enum : int { kOk = 0, kOverflow = 1, kCapacity = 2 };
// error bits of the context's device flag (read back by sync calls)
enum : int { kErrPlanCapacity = 1, kErrParticleCapacity = 2, kErrInternal = 16 };

struct StepParams {
  int model, adaptive, m_fixed, m_cap, indicator, log_on;
  double alpha;            // VHS exponent
  int wb, wb_max;          // TRMC-WB definition (0 off) and threshold
  int sigma_update;        // majorant raised after each proposal [R33]
  double delta1, delta2, dt, eps;
  uint32_t k0, k1, step, cell_base;
  int shock;               // rho_c = n w / dx when 1, else 1
  double w_over_dx;
  int *err;                // device error bits
  int debug_stop;          // debug: >0 stops after that many RAD retries (no Maxwellian)
};

// Per-CTA working set.  Index type: uint32.
template <typename Real>
struct CellBuf {
  Real *vx, *vy, *vz;      // [n] cell velocities (smem copy or global, in place)
  uint32_t *ctype;         // [K_cap] type a of collision (level d, j) at S[d]+j
  uint32_t *crank;         // [K_cap] rank among same-type collisions of its level
  uint32_t *cslot;         // [2 K_cap] input/output slots (side 0, side 1)
  uint8_t *ctype8;         // warp kernel: compact copies of the three above (types < 256,
  uint16_t *crank16;       //   ranks and slots < 65536), so more warps fit an SM
  uint16_t *cslot16;
  int32_t *Q;              // [L_cap+1] split quotas N_d
  int32_t *C;              // [L_cap+1] collisions per level
  int32_t *S;              // [L_cap+1] first collision index of level
  int32_t *cons;           // [L_cap+1] demands on pool d
  int32_t *base;           // [L_cap+1] running demand counter of pool d
  int32_t *cnt;            // [L_cap+1] per-type counter of the current level
  uint4 *rk;               // [L_cap+1] permutation keys of pools
  uint32_t *mask;          // [ceil(n_cap/32)] Theta membership
  PermDom *pdom;           // [L_cap+1] warp kernel: domain of pool p's permutation (or null)
  double *wlen;            // [K_cap] TRMC-WB: tree length of collision k's outputs (or null)
  uint8_t *wused;          // [2 K_cap] TRMC-WB: output o consumed by a higher level
  double *red;             // [32*8] reduction scratch
  int n_cap, K_cap, L_cap;
};

constexpr int kSplitPre = 72;
// Scalars shared by the CTA.
struct CellShared {
  double ux, uy, uz, S0, sigma, p, mu, S_est, E1;
  double sig_run;             // running majorant (sigma_update) [R33]
  double sums[8];
  int n, m, m_cur, m_next, d, top, lo, hi, r, planned, flag, done;
  int64_t rem;
  int32_t L, Ltot, U, nT, budget, leaf_off, attempts, ktot, nwb;
  int32_t solo_from, cnt_d, cnt_S;   // grid team: levels small enough for block 0 alone
  unsigned long long prop, acc, viol;
  double usplit[kSplitPre];   // split uniforms of levels < kSplitPre, drawn in parallel
};

template <typename Real> struct RealOps;
template <> struct RealOps<double> {
  __device__ static __forceinline__ double sqrt_(double x) { return sqrt(x); }
  __device__ static __forceinline__ void sincospi_(double x, double *s, double *c) { sincospi(x, s, c); }
  __device__ static __forceinline__ double pow_(double x, double a) { return pow(x, a); }
};
template <> struct RealOps<float> {
  __device__ static __forceinline__ float sqrt_(float x) { return sqrtf(x); }
  __device__ static __forceinline__ void sincospi_(float x, float *s, float *c) { sincospif(x, s, c); }
  __device__ static __forceinline__ float pow_(float x, float a) { return powf(x, a); }
};

// VHS majorant Sigma' = (2 sqrt(dv2))^alpha (Sigma = sigma(2 dv); K cancels).
__device__ __forceinline__ double vhs_majorant(double dv2, double alpha) { return pow(2.0 * sqrt(dv2), alpha); }

// TRMC-WB tree length of a level-d collision's outputs from its inputs'
// lengths a, b (samples of f_0: 0): eq. def:2 (1 + min), def:3 (1 + mean),
// def:1 (d).  Same arithmetic as the oracle (exact dyadic sums in fp64).
__device__ __forceinline__ double wb_combine(int def, int d, double a, double b) {
  if (def == 1) return 1.0 + (a < b ? a : b);
  if (def == 2) return 1.0 + 0.5 * (a + b);
  return (double)d;
}

// IR at split level d with its keyed uniform; exact 0 when y < 2^-53.
// Uniforms of levels < kSplitPre were drawn in parallel into `pre`.
__device__ __forceinline__ int64_t ir_split(const RngKey &K, int d, double y, const double *pre,
                                            int npre = kSplitPre) {
  if (y < 0x1p-53) return 0;
  double u;
  if (d < npre) {
    u = pre[d];
  } else {
    const uint4 w = K(kSplit, 0, (uint32_t)d, 0);
    u = u53(w.x, w.y);
  }
  const double fl = floor(y);
  return (int64_t)fl + ((u < y - fl) ? 1 : 0);
}

// Alg 4.2 continued until rem == 0 or level m (thread 0 only).  Quotas above
// L_cap cannot be stored: a non-zero one flags overflow.
__device__ inline void split_extend(const RngKey &K, CellShared &sh, int m, int32_t *Q, int L_cap) {
  while (sh.rem > 0 && sh.d < m) {
    const double y = sh.p * (double)sh.rem;
    if (y < 0x1p-53) {                     // every further IR is exactly 0
      for (int d = sh.d + 1; d <= m && d <= L_cap; ++d) Q[d] = 0;
      sh.d = m;
      break;
    }
    sh.d++;
    int64_t q = ir_split(K, sh.d, y, sh.usplit);
    if (q > sh.rem) q = sh.rem;
    if (sh.d <= L_cap) Q[sh.d] = (int32_t)q;
    else if (q > 0) sh.flag = kOverflow;
    sh.rem -= q;
  }
}

template <typename Real>
__device__ __forceinline__ void load3(const Real *a, const Real *b, const Real *c, int64_t i, Real &x,
                                      Real &y, Real &z) {
  x = a[i]; y = b[i]; z = c[i];
}

// (qx^2 + qy^2) + qz^2 and |q|, every product and sum rounded (no FMA
// contraction: the oracle's order, and the same value wherever it is taken;
// for a two-particle cell |q| and Sigma' = 2 max|v - u| tie mathematically)
__device__ __forceinline__ double sq3(double qx, double qy, double qz) {
  return __dadd_rn(__dadd_rn(__dmul_rn(qx, qx), __dmul_rn(qy, qy)), __dmul_rn(qz, qz));
}
__device__ __forceinline__ double qnorm(double qx, double qy, double qz) { return sqrt(sq3(qx, qy, qz)); }
__device__ __forceinline__ float qnorm(float qx, float qy, float qz) {
  return sqrtf(__fadd_rn(__fadd_rn(__fmul_rn(qx, qx), __fmul_rn(qy, qy)), __fmul_rn(qz, qz)));
}

// A violation is a pair above the bound by more than the bound's own rounding
// [R35]: in a two-particle cell |q| = 2 max|v - u| exactly, and a strict
// comparison would count rounding noise.  Sigma' (1 + 2^-40) in fp64,
// Sigma' (1 + 2^-20) in fp32 (the oracle: the fp64 one).
__device__ __forceinline__ double viol_bound(double s) { return s * (1.0 + 0x1p-40); }
__device__ __forceinline__ float viol_bound(float s) { return s * (1.0f + 0x1p-20f); }

// sigma_ij / K of the pair in slots (si, sk): |q| (HS) or |q|^alpha (VHS).
// Used by the majorant variant [R33] to find a level's largest proposal.
template <typename Real>
__device__ __forceinline__ Real pair_sigma(const StepParams &P, const CellBuf<Real> &B, uint32_t si, uint32_t sk) {
  const Real q = qnorm(B.vx[si] - B.vx[sk], B.vy[si] - B.vy[sk], B.vz[si] - B.vz[sk]);
  return P.model == TRMCR_VHS ? RealOps<Real>::pow_(q, (Real)P.alpha) : q;
}

// A6 on the pair in slots (si, sk) of (vx, vy, vz) with the collision's
// uniforms: acceptance against the bound (dummy collision when rejected),
// then v' = G +- (|q|/2) sigma.  Returns accepted.
// RAD indicator of one velocity (R20): (v_x - u_x)^2 (Pxx) or |v|^4 (M4).
template <typename Real>
__device__ __forceinline__ Real ind_value(bool pxx, Real ux, Real x, Real y, Real z) {
  if (pxx) { const Real dx = x - ux; return dx * dx; }
  const Real v2 = x * x + y * y + z * z;
  return v2 * v2;
}

// dS (nullable): an accepted collision adds the change of the cell's indicator
// sum, ind(a') + ind(b') - ind(a) - ind(b), so the RAD estimate needs no pass
// over the whole cell (warp kernels; the sum telescopes over a slot's
// successive collisions).
// MOD >= 0: the collision model fixed at compile time (the hard-sphere
// instantiation of the shock kernel carries no VHS / Maxwell code); -1: P.model.
template <typename Real, int MOD = -1>
__device__ __forceinline__ int pair_collide(const StepParams &P, Real *vx, Real *vy, Real *vz, Real sigma,
                                            Real xa, Real xi1, Real xi2, uint32_t si, uint32_t sk,
                                            unsigned &viol, double *dS = nullptr, Real ind_ux = Real(0)) {
  using O = RealOps<Real>;
  const Real ax = vx[si], ay = vy[si], az = vz[si];
  const Real bx = vx[sk], by = vy[sk], bz = vz[sk];
  const Real q = qnorm(ax - bx, ay - by, az - bz);
  const int model = MOD >= 0 ? MOD : P.model;
  int acc = 1;
  if (model == TRMCR_HARD_SPHERE) {         // accept iff xi Sigma' < |q|  [R7]
    viol += (q > viol_bound(sigma)) ? 1u : 0u;
    acc = (xa * sigma < q);
  } else if (model == TRMCR_VHS) {          // accept iff xi Sigma' < |q|^alpha (sec. VHS)
    const Real qa = O::pow_(q, (Real)P.alpha);
    viol += (qa > viol_bound(sigma)) ? 1u : 0u;
    acc = (xa * sigma < qa);
  }
  if (acc) {
    const Real c = Real(2) * xi1 - Real(1);
    const Real s = O::sqrt_((Real(1) - c) * (Real(1) + c));
    Real sp, cp;
    O::sincospi_(Real(2) * xi2, &sp, &cp);
    const Real h = Real(0.5) * q;
    const Real hx = h * (s * cp), hy = h * (s * sp), hz = h * c;
    const Real gx = Real(0.5) * (ax + bx), gy = Real(0.5) * (ay + by), gz = Real(0.5) * (az + bz);
    const Real nax = gx + hx, nay = gy + hy, naz = gz + hz, nbx = gx - hx, nby = gy - hy, nbz = gz - hz;
    vx[si] = nax; vy[si] = nay; vz[si] = naz;
    vx[sk] = nbx; vy[sk] = nby; vz[sk] = nbz;
    if (dS) {
      const bool pxx = P.indicator == TRMCR_IND_PXX;
      const Real dn = ind_value<Real>(pxx, ind_ux, nax, nay, naz) + ind_value<Real>(pxx, ind_ux, nbx, nby, nbz);
      const Real dold = ind_value<Real>(pxx, ind_ux, ax, ay, az) + ind_value<Real>(pxx, ind_ux, bx, by, bz);
      *dS += (double)(dn - dold);
    }
  }
  return acc;
}

// One (dummy) collision of a tree node (A6) with its keyed draws
// (COLL, attempt, level, j).  Returns accepted.
template <typename Real, int MOD = -1>
__device__ __forceinline__ int tree_collision(const StepParams &P, const RngKey &K, CellBuf<Real> &B,
                                              Real sigma, int r, int d, uint32_t j, uint32_t si,
                                              uint32_t sk, unsigned &viol, double *dS = nullptr,
                                              Real ind_ux = Real(0)) {
  Real xa, xi1, xi2;
  if constexpr (sizeof(Real) == 8) {
    const uint4 w = K(kColl, r, d, j);
    const uint4 w2 = K(kColl2, r, d, j);
    xa = u53(w.x, w.y); xi1 = u53(w.z, w.w); xi2 = u53(w2.x, w2.y);
  } else {
    const uint4 w = K(kColl, r, d, j);
    xa = u24(w.x); xi1 = u24(w.y); xi2 = u24(w.z);
  }
  return pair_collide<Real, MOD>(P, B.vx, B.vy, B.vz, sigma, xa, xi1, xi2, si, sk, viol, dS, ind_ux);
}

// Draw three standard normals for Theta slot `slot` (Box-Muller).
template <typename Real>
__device__ __forceinline__ void gauss3(const RngKey &K, uint32_t slot, Real &g0, Real &g1, Real &g2) {
  if constexpr (sizeof(Real) == 8) {
    const uint4 w = K(kMaxw, 0, 0, slot);
    const uint4 w2 = K(kMaxw2, 0, 0, slot);
    const double u1 = u53(w.x, w.y), u2 = u53(w.z, w.w), u3 = u53(w2.x, w2.y), u4 = u53(w2.z, w2.w);
    const double r1 = sqrt(-2.0 * log(u1)), r3 = sqrt(-2.0 * log(u3));
    double s2, c2, s4, c4;
    sincospi(2.0 * u2, &s2, &c2);
    sincospi(2.0 * u4, &s4, &c4);
    g0 = r1 * c2; g1 = r1 * s2; g2 = r3 * c4;
  } else {
    const uint4 w = K(kMaxw, 0, 0, slot);
    const float u1 = u24(w.x), u2 = u24(w.y), u3 = u24(w.z), u4 = u24(w.w);
    const float r1 = sqrtf(-2.0f * __logf(u1)), r3 = sqrtf(-2.0f * __logf(u3));
    float s2, c2;
    __sincosf(6.283185307179586f * u2, &s2, &c2);
    const float c4 = __cosf(6.283185307179586f * u4);
    g0 = r1 * c2; g1 = r1 * s2; g2 = r3 * c4;
  }
}

// ---------------------------------------------------------------------------
// Plan (A5), top-down: C_d = ceil((Q_d + cons_d)/2) collisions per level,
// each with a type a uniform in {0..d-1} consuming one sample of f_a
// and one of f_{d-1-a}.  Quotas only on [lo, hi].  Guard: if the
// leaves cons_0 exceed `budget`, drop the top quota level and re-plan.
// ---------------------------------------------------------------------------
// ---- execution teams of the CTA-level step code: one CTA (BlockTeam), or
// the whole grid of a cooperative launch (GridTeam: one giant cell on every
// SM).  tid/size/sync/reductions are the team's; reductions are two-level
// and in a fixed order (deterministic). ----
constexpr int kGridSlots = 8;
// Levels with fewer collisions than this run on block 0 alone ("solo": CTA
// barriers instead of grid barriers; the rest of the grid waits at the next
// grid barrier) - a grid barrier costs more than such a level's work.
constexpr int kSoloMax = 2048;
struct GridTeam {
  static constexpr bool kGrid = true;
  double *part;              // [kGridSlots][gridDim.x][8] per-block partial sums (rotating)
  int32_t *hbuf;             // rank scratch [hcap]
  int64_t hcap;
  int slot;
  bool solo = false;         // block 0 alone (tid/size/sync/reductions of the CTA)
  __device__ __forceinline__ int tid() const { return solo ? (int)threadIdx.x : blockIdx.x * blockDim.x + threadIdx.x; }
  __device__ __forceinline__ int size() const { return solo ? (int)blockDim.x : gridDim.x * blockDim.x; }
  // cooperative-groups grid barrier: release/acquire at gpu scope, so plain
  // loads after it see every write made before it
  __device__ __forceinline__ void sync() const {
    if (solo) __syncthreads();
    else cooperative_groups::this_grid().sync();
  }
  template <int NV> __device__ void sum(double (&v)[NV], double *red) {
    static_assert(NV <= 8, "at most 8 sums");
    block_sum<NV>(v, red);
    if (solo) return;
    double *pp = part + (size_t)slot * gridDim.x * 8;
    if (threadIdx.x == 0)
      for (int k = 0; k < NV; ++k) pp[blockIdx.x * 8 + k] = v[k];
    sync();
    for (int k = 0; k < NV; ++k) {
      double t = 0.0;
      for (int b = 0; b < (int)gridDim.x; ++b) t += pp[b * 8 + k];   // block order: deterministic
      v[k] = t;
    }
    slot = (slot + 1) % kGridSlots;
  }
  __device__ double max(double x, double *red) {
    x = block_max(x, red);
    if (solo) return x;
    double *pp = part + (size_t)slot * gridDim.x * 8;
    if (threadIdx.x == 0) pp[blockIdx.x * 8] = x;
    sync();
    double t = 0.0;
    for (int b = 0; b < (int)gridDim.x; ++b) t = fmax(t, pp[b * 8]);
    slot = (slot + 1) % kGridSlots;
    return t;
  }
};

struct BlockTeam {
  static constexpr bool kGrid = false;
  bool solo = false;
  int32_t *hbuf = nullptr;   // no separate rank scratch (the level's slot range is used)
  int64_t hcap = 0;
  __device__ __forceinline__ int tid() const { return threadIdx.x; }
  __device__ __forceinline__ int size() const { return blockDim.x; }
  __device__ __forceinline__ void sync() const { __syncthreads(); }
  template <int NV> __device__ __forceinline__ void sum(double (&v)[NV], double *red) { block_sum<NV>(v, red); }
  __device__ __forceinline__ double max(double x, double *red) { return block_max(x, red); }
};

template <typename Real, class Team>
__device__ void plan_counts(Team &T, const RngKey &K, CellBuf<Real> &B, CellShared &sh) {
  const int tid = T.tid();
  if (tid == 0) {
    int top = sh.hi;
    while (top >= sh.lo && B.Q[top] == 0) top--;
    sh.top = top;
    sh.planned = 0;
    sh.done = 0;
  }
  T.sync();
  for (;;) {
    if (sh.top < sh.lo || sh.top < 1) {    // nothing to plan
      if (tid == 0) { sh.top = 0; sh.L = 0; }
      T.sync();
      return;
    }
    if (sh.top > B.L_cap) {
      if (tid == 0) sh.flag = kOverflow;
      T.sync();
      return;
    }
    const int top = sh.top;
    for (int d = tid; d <= top; d += T.size()) B.cons[d] = 0;
    T.sync();
    int Sacc = 0;
    int d = top;
    if constexpr (Team::kGrid) {
      // the small top levels on block 0 alone, up to the first large one
      if (blockIdx.x == 0) {
        T.solo = true;
        const int t0 = T.tid();
        for (; d >= 1; --d) {
          const int Qd = (d >= sh.lo) ? B.Q[d] : 0;
          const int Cd = (Qd + B.cons[d] + 1) >> 1;
          if (Cd >= kSoloMax) break;
          if ((int64_t)Sacc + Cd > B.K_cap) { d = -1; break; }
          if (t0 == 0) { B.C[d] = Cd; B.S[d] = Sacc; }
          for (int j = t0; j < Cd; j += T.size()) {
            const uint32_t w = K(kType, sh.r, d, j).x;
            const uint32_t a = __umulhi(w, (uint32_t)d);
            B.ctype[Sacc + j] = a;
            const unsigned act = __activemask();
            const unsigned pa = __match_any_sync(act, a), pb = __match_any_sync(act, (uint32_t)d - 1u - a);
            const int lane_ = threadIdx.x & 31;
            if ((__ffs(pa) - 1) == lane_) atomicAdd(&B.cons[a], __popc(pa));
            if ((__ffs(pb) - 1) == lane_) atomicAdd(&B.cons[d - 1 - a], __popc(pb));
          }
          Sacc += Cd;
          T.sync();
        }
        T.solo = false;
        if (t0 == 0) {
          sh.cnt_d = d; sh.cnt_S = Sacc;
          if (d < 0) sh.flag = kOverflow;
        }
      }
      T.sync();
      d = sh.cnt_d;
      Sacc = sh.cnt_S;
      if (d < 0) return;
    }
    for (; d >= 1; --d) {
      const int Qd = (d >= sh.lo) ? B.Q[d] : 0;
      const int Cd = (Qd + B.cons[d] + 1) >> 1;   // all threads read the same value
      if ((int64_t)Sacc + Cd > B.K_cap) {
        T.sync();
        if (tid == 0) sh.flag = kOverflow;
        T.sync();
        return;
      }
      // (no barrier here: level d's draws only add to cons[a < d], never to the
      // cons[d] every thread has just read; the end-of-level barrier orders levels)
      if (tid == 0) { B.C[d] = Cd; B.S[d] = Sacc; }
      for (int j = tid; j < Cd; j += T.size()) {
        const uint32_t w = K(kType, sh.r, d, j).x;
        const uint32_t a = __umulhi(w, (uint32_t)d);  // floor(w d / 2^32)
        B.ctype[Sacc + j] = a;
        // warp-aggregated demand counts (one atomic per distinct pool per warp)
        const unsigned act = __activemask();
        const unsigned pa = __match_any_sync(act, a), pb = __match_any_sync(act, (uint32_t)d - 1u - a);
        const int lane_ = threadIdx.x & 31;
        if ((__ffs(pa) - 1) == lane_) atomicAdd(&B.cons[a], __popc(pa));
        if ((__ffs(pb) - 1) == lane_) atomicAdd(&B.cons[d - 1 - a], __popc(pb));
      }
      Sacc += Cd;
      T.sync();
    }
    if (tid == 0) {
      if (B.cons[0] <= sh.budget) {
        sh.L = B.cons[0];
        sh.done = 1;
      } else {                                    // drop the top quota level
        int t = sh.top - 1;
        while (t >= sh.lo && B.Q[t] == 0) t--;
        sh.top = t;
      }
    }
    T.sync();
    if (sh.done) return;
  }
}

// Decision-log record of one collision (parity mode).
__device__ __forceinline__ void log_collision(const StepParams &P, const RngKey &K, trmcr_coll_rec *log,
                                              unsigned long long *log_count, int64_t log_cap, int r, int d,
                                              int j, int ok, uint32_t s0, uint32_t s1) {
  if (!P.log_on) return;
  const unsigned long long at = atomicAdd(log_count, 1ull);
  if ((int64_t)at < log_cap) {
    trmcr_coll_rec rec;
    rec.cell = (int32_t)K.cell; rec.attempt = r; rec.level = d; rec.accepted = ok;
    rec.j = j; rec.slot_i = s0; rec.slot_k = s1;
    log[at] = rec;
  }
}

// Bottom-up slot resolution + execution (A5, A6): level d's demand on pool p
// has rank base_p + (in-level rank); side-0 demands (type p) precede side-1
// demands (type d-1-p).  Pool p's t-th demand takes output pi_p(t) of level
// p (pi_0 = leaf order of the cell).  Output side s of a collision keeps the
// slot of its input side s; collisions of one level touch disjoint slots.
template <typename Real, class Team>
__device__ void plan_execute(Team &T, const StepParams &P, const RngKey &K, CellBuf<Real> &B, CellShared &sh,
                             const Perm &pi0, Real sigma, trmcr_coll_rec *log,
                             unsigned long long *log_count, int64_t log_cap) {
  const int tid = T.tid(), lane = tid & 31, warp = tid >> 5;
  const int top = sh.top;
  if (top < 1) return;
  for (int d = tid; d <= top; d += T.size()) {
    B.base[d] = 0;
    B.cnt[d] = 0;
    if (d >= 1) B.rk[d] = K(kPerm, sh.r, d, 0);
  }
  const int ktot = B.S[1] + B.C[1];                // collisions of the plan (levels top..1 stored from 0)
  if (P.wb) for (int o = tid; o < 2 * ktot; o += T.size()) B.wused[o] = 0;
  if (tid == 0) {
    sh.ktot = ktot;
    int sf = top + 1;                               // levels >= sf are all small
    while (sf > 1 && B.C[sf - 1] < kSoloMax) --sf;
    sh.solo_from = sf;
  }
  if (T.hbuf) {            // grid team: the large levels' rank scratch starts zeroed
    const int64_t hz = min((int64_t)(T.size() >> 5) * top, T.hcap);
    for (int64_t q = tid; q < hz; q += T.size()) T.hbuf[q] = 0;
  }
  T.sync();
  const int solo_from = sh.solo_from;
  unsigned acc = 0, viol = 0;
  const int r = sh.r;
  const int leaf_off = sh.leaf_off;
  int pd = 0;            // last level with collisions: its histogram is still in cnt[]
  for (int d = 1; d <= top; ++d) {
    if constexpr (Team::kGrid) {
      if (!T.solo && d >= solo_from) {     // the remaining levels are small: block 0 alone
        if (blockIdx.x != 0) break;
        T.solo = true;
      }
    }
    const int Cd = B.C[d], Sd = B.S[d];
    if (Cd == 0) continue;
    const int nw = T.size() >> 5;
    // large levels: ranks by all warps (chunk histograms in the level's own,
    // not yet written, cslot range: nw * d ints <= 2 Cd; a grid team has its
    // own scratch)
    const bool par = Cd >= 2048 && (T.hbuf ? (int64_t)nw * d <= T.hcap : nw * d <= 2 * Cd);
    if (warp == 0) {
      // fold level pd's demands into base[] and clear its histogram (cnt)
      // (two passes through cons[], idle during execution: every read of the
      // histogram happens before any of it is cleared)
      if (pd > 0) {
        for (int p = lane; p < pd; p += 32) B.cons[p] = B.base[p] + B.cnt[p] + B.cnt[pd - 1 - p];
        __syncwarp();
        for (int p = lane; p < pd; p += 32) { B.base[p] = B.cons[p]; B.cnt[p] = 0; }
        __syncwarp();
      }
    }
    if (par) {
      // same ranks as the serial loop below: warp w owns collisions
      // [w chunk, (w + 1) chunk); H[w][a] = its count of type a, then the
      // exclusive prefix over warps, then the in-order walk
      int32_t *H = T.hbuf ? T.hbuf : reinterpret_cast<int32_t *>(B.cslot + 2 * (size_t)Sd);
      const int chunk = (Cd + nw - 1) / nw;
      if (!T.hbuf) {          // a grid team's scratch is kept zeroed between levels
        for (int q = tid; q < nw * d; q += T.size()) H[q] = 0;
        T.sync();
      }
      const int j_lo = warp * chunk, j_hi = min(Cd, j_lo + chunk);
      for (int j0 = j_lo; j0 < j_hi; j0 += 32) {
        const int j = j0 + lane;
        const bool valid = j < j_hi;
        const uint32_t a = valid ? B.ctype[Sd + j] : 0xFFFFFFFFu;
        const unsigned peers = __match_any_sync(0xffffffffu, a);
        if (valid && (__ffs(peers) - 1) == lane) H[warp * d + (int)a] += __popc(peers);
        __syncwarp();
      }
      T.sync();
      for (int t = tid; t < d; t += T.size()) {
        int run = 0;
        for (int w = 0; w < nw; ++w) { const int v = H[w * d + t]; H[w * d + t] = run; run += v; }
        B.cnt[t] = run;                       // the level's type histogram
      }
      T.sync();
      for (int j0 = j_lo; j0 < j_hi; j0 += 32) {
        const int j = j0 + lane;
        const bool valid = j < j_hi;
        const uint32_t a = valid ? B.ctype[Sd + j] : 0xFFFFFFFFu;
        const unsigned peers = __match_any_sync(0xffffffffu, a);
        const unsigned lt = (1u << lane) - 1u;
        int c0 = 0;
        if (valid) c0 = H[warp * d + (int)a];
        __syncwarp();
        if (valid) {
          B.crank[Sd + j] = (uint32_t)(c0 + __popc(peers & lt));
          if ((peers & lt) == 0u) H[warp * d + (int)a] = c0 + __popc(peers);
        }
        __syncwarp();
      }
    } else if (warp == 0) {
      // in-level stable ranks per type (32 collisions per round); cnt ends as
      // this level's type histogram
      for (int j0 = 0; j0 < Cd; j0 += 32) {
        const int j = j0 + lane;
        const bool valid = j < Cd;
        const uint32_t a = valid ? B.ctype[Sd + j] : 0xFFFFFFFFu;
        const unsigned peers = __match_any_sync(0xffffffffu, a);
        const unsigned lt = (1u << lane) - 1u;
        int c0 = 0;
        if (valid) c0 = B.cnt[a];
        __syncwarp();
        if (valid) {
          B.crank[Sd + j] = (uint32_t)(c0 + __popc(peers & lt));
          if ((peers & lt) == 0u) B.cnt[a] = c0 + __popc(peers);
        }
        __syncwarp();
      }
    }
    pd = d;
    T.sync();
    for (int j = tid; j < Cd; j += T.size()) {
      const uint32_t a = B.ctype[Sd + j], b = (uint32_t)d - 1u - a;
      const uint32_t rank = B.crank[Sd + j];
      const uint32_t t[2] = {(uint32_t)B.base[a] + rank, (uint32_t)(B.base[b] + B.cnt[b]) + rank};
      const uint32_t pool[2] = {a, b};
      uint32_t slot[2];
      double ln[2] = {0.0, 0.0};             // TRMC-WB input lengths (samples of f_0: 0)
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        if (pool[s] == 0) {
          slot[s] = pi0((uint32_t)leaf_off + t[s]);
        } else {
          Perm pp;
          pp.init(B.rk[pool[s]], 2u * (uint32_t)B.C[pool[s]]);
          const uint32_t o = pp(t[s]);
          slot[s] = o == 0xFFFFFFFFu ? o : B.cslot[2u * (uint32_t)B.S[pool[s]] + o];
          if (P.wb && o != 0xFFFFFFFFu) {
            const uint32_t og = 2u * (uint32_t)B.S[pool[s]] + o;
            B.wused[og] = 1;
            ln[s] = B.wlen[og >> 1];
          }
        }
        if (slot[s] >= (uint32_t)sh.n) {   // cannot happen: internal fault, never hang
          atomicOr(P.err, kErrInternal);
          slot[s] = 0;
        }
      }
      B.cslot[2 * (Sd + j)] = slot[0];
      B.cslot[2 * (Sd + j) + 1] = slot[1];
      if (P.wb) B.wlen[Sd + j] = wb_combine(P.wb, d, ln[0], ln[1]);
      if (!P.sigma_update) {
        const int ok = tree_collision<Real>(P, K, B, sigma, r, d, (uint32_t)j, slot[0], slot[1], viol);
        acc += ok;
        log_collision(P, K, log, log_count, log_cap, r, d, j, ok, slot[0], slot[1]);
      }
    }
    if (P.sigma_update) {
      // majorant raised after each proposal [R33]: the level's collisions are
      // independent, so if none of them exceeds the running bound they all
      // run in parallel with it; otherwise one thread runs the level in
      // canonical order, raising the bound as it goes (rare: violations)
      T.sync();
      double mx = 0.0;
      for (int j = tid; j < Cd; j += T.size())
        mx = fmax(mx, (double)pair_sigma<Real>(P, B, B.cslot[2 * (Sd + j)], B.cslot[2 * (Sd + j) + 1]));
      mx = T.max(mx, B.red);
      if (mx > (double)viol_bound(sigma)) {
        if (tid == 0) {
          for (int j = 0; j < Cd; ++j) {
            const uint32_t s0 = B.cslot[2 * (Sd + j)], s1 = B.cslot[2 * (Sd + j) + 1];
            const Real sj = pair_sigma<Real>(P, B, s0, s1);
            const int ok = tree_collision<Real>(P, K, B, sigma, r, d, (uint32_t)j, s0, s1, viol);
            acc += ok;
            log_collision(P, K, log, log_count, log_cap, r, d, j, ok, s0, s1);
            if (sj > viol_bound(sigma)) sigma = sj;
          }
          sh.sig_run = (double)sigma;
        }
        T.sync();
        sigma = (Real)sh.sig_run;
      } else {
        for (int j = tid; j < Cd; j += T.size()) {
          const uint32_t s0 = B.cslot[2 * (Sd + j)], s1 = B.cslot[2 * (Sd + j) + 1];
          const int ok = tree_collision<Real>(P, K, B, sigma, r, d, (uint32_t)j, s0, s1, viol);
          acc += ok;
          log_collision(P, K, log, log_count, log_cap, r, d, j, ok, s0, s1);
        }
      }
    }
    if (tid == 0) sh.prop += (unsigned long long)Cd;
    if (par && T.hbuf)     // re-zero the rank scratch for the next large level (no barrier of its own)
      for (int q = tid; q < nw * d; q += T.size()) T.hbuf[q] = 0;
    T.sync();
  }
  T.solo = false;        // every block meets at the grid barrier below
  atomicAdd(&sh.acc, (unsigned long long)acc);
  atomicAdd(&sh.viol, (unsigned long long)viol);
  T.sync();
}

// RAD indicator estimate with Theta taken analytically:
// S_est = [sum over the non-Theta particles + |Theta| (analytic Maxwellian
// term)] / n.  Theta's particles are still their pre-step values, so the
// non-Theta sum is (sum over all slots) - (sum over Theta's slots): one pass
// over the cell plus one over Theta's slots, no membership table.
template <typename Real, class Team>
__device__ void rad_estimate(Team &T, const StepParams &P, CellBuf<Real> &B, CellShared &sh, const Perm &pi0) {
  const int tid = T.tid(), n = sh.n, nT = sh.nT;
  const bool pxx = P.indicator == TRMCR_IND_PXX;
  double v[8] = {0, 0, 0, 0, 0, 0, 0, 0};   // all-slot indicator sum; Theta: indicator, momentum, |v|^2
  for (int i = tid; i < n; i += T.size()) {
    const double x = B.vx[i], y = B.vy[i], z = B.vz[i];
    if (pxx) {
      const double dx = x - sh.ux;
      v[0] += dx * dx;
    } else {
      const double v2 = x * x + y * y + z * z;
      v[0] += v2 * v2;
    }
  }
  for (int q = tid; q < nT; q += T.size()) {
    const uint32_t s = pi0((uint32_t)(sh.Ltot + q));
    if (s >= (uint32_t)n) { atomicOr(P.err, kErrInternal); continue; }
    const double x = B.vx[s], y = B.vy[s], z = B.vz[s];
    if (pxx) {
      const double dx = x - sh.ux;
      v[1] += dx * dx;
    } else {
      const double v2 = x * x + y * y + z * z;
      v[1] += v2 * v2;
    }
    v[2] += x; v[3] += y; v[4] += z;
    v[5] += x * x + y * y + z * z;
  }
  T.template sum<6>(reinterpret_cast<double(&)[6]>(v), B.red);
  if (tid == 0) {
    double s = v[0] - v[1];
    if (nT > 0) {
      const double tx = v[2] / nT, ty = v[3] / nT, tz = v[4] / nT;
      const double T = fmax(0.0, v[5] / nT - (tx * tx + ty * ty + tz * tz)) / 3.0;
      if (pxx) {
        s += (double)nT * (T + (tx - sh.ux) * (tx - sh.ux));
      } else {
        const double u2 = tx * tx + ty * ty + tz * tz;
        s += (double)nT * (u2 * u2 + 10.0 * u2 * T + 15.0 * T * T);
      }
    }
    sh.S_est = s / n;
    if (sh.S0 != 0.0) sh.E1 = fabs(sh.S_est - sh.S0) / fabs(sh.S0);
    else sh.E1 = (sh.S_est == 0.0) ? 0.0 : INFINITY;
  }
  T.sync();
}

// Conservative Maxwellian (A8) over Theta = pi0 positions [Ltot, Ltot+nT)
// plus, under TRMC-WB, the final outputs whose tree is longer than wb_max
// (index q < nT: pi0(Ltot + q); q >= nT: output q - nT of the plan).
template <typename Real, class Team>
__device__ void maxwellian(Team &T, const StepParams &P, const RngKey &K, CellBuf<Real> &B, CellShared &sh,
                           const Perm &pi0, double ec_all) {
  const int tid = T.tid(), nT = sh.nT;
  const int nq = nT + (P.wb ? 2 * sh.ktot : 0);
  auto member = [&](int q, uint32_t &s) -> bool {
    if (q < nT) { s = pi0((uint32_t)(sh.Ltot + q)); return true; }
    const int o = q - nT;
    if (B.wused[o] || !(B.wlen[o >> 1] > (double)P.wb_max)) return false;
    s = B.cslot[o];
    return true;
  };
  int nwb = 0;
  if (P.wb) {
    double c1[1] = {0.0};
    for (int o = tid; o < 2 * sh.ktot; o += T.size())
      c1[0] += (!B.wused[o] && B.wlen[o >> 1] > (double)P.wb_max) ? 1.0 : 0.0;
    T.template sum<1>(c1, B.red);
    nwb = (int)c1[0];
  }
  if (tid == 0) sh.nwb = nwb;
  const int nTT = nT + nwb;
  if (nTT < 2) { T.sync(); return; }
  const bool full = (nT == sh.n);          // Theta = every slot: skip the permutation
  double ux, uy, uz, ec;
  if (full) {
    ux = sh.ux; uy = sh.uy; uz = sh.uz; ec = ec_all;
  } else {
    double v[3] = {0, 0, 0};
    for (int q = tid; q < nq; q += T.size()) {
      uint32_t s;
      if (!member(q, s)) continue;
      if (s >= (uint32_t)sh.n) { atomicOr(P.err, kErrInternal); continue; }
      v[0] += (double)B.vx[s]; v[1] += (double)B.vy[s]; v[2] += (double)B.vz[s];
    }
    T.template sum<3>(v, B.red);
    ux = v[0] / nTT; uy = v[1] / nTT; uz = v[2] / nTT;
    ec = 0;
  }
  double g[5] = {0, 0, 0, 0, 0};   // sum g (3), sum |g|^2, centred energy of Theta
  for (int q = tid; q < nq; q += T.size()) {
    uint32_t s = (uint32_t)q;
    if (!full && !member(q, s)) continue;
    if (s >= (uint32_t)sh.n) { atomicOr(P.err, kErrInternal); continue; }
    if (!full) {
      const double dx = B.vx[s] - ux, dy = B.vy[s] - uy, dz = B.vz[s] - uz;
      g[4] += dx * dx + dy * dy + dz * dz;
    }
    Real g0, g1, g2;
    gauss3<Real>(K, s, g0, g1, g2);
    B.vx[s] = g0; B.vy[s] = g1; B.vz[s] = g2;   // park g in place (same thread rewrites)
    g[0] += g0; g[1] += g1; g[2] += g2;
    g[3] += (double)g0 * g0 + (double)g1 * g1 + (double)g2 * g2;
  }
  T.template sum<5>(g, B.red);
  if (!full) ec = g[4];
  const double gx = g[0] / nTT, gy = g[1] / nTT, gz = g[2] / nTT;
  const double D = g[3] - nTT * (gx * gx + gy * gy + gz * gz);
  const double sc = (D > 0.0 && ec > 0.0) ? sqrt(ec / D) : 0.0;
  const Real rsc = (Real)sc, rgx = (Real)gx, rgy = (Real)gy, rgz = (Real)gz;
  const Real rux = (Real)ux, ruy = (Real)uy, ruz = (Real)uz;
  for (int q = tid; q < nq; q += T.size()) {
    uint32_t s = (uint32_t)q;
    if (!full && !member(q, s)) continue;
    if (s >= (uint32_t)sh.n) continue;
    B.vx[s] = rux + rsc * (B.vx[s] - rgx);
    B.vy[s] = ruy + rsc * (B.vy[s] - rgy);
    B.vz[s] = ruz + rsc * (B.vz[s] - rgz);
  }
  T.sync();
}

// Full per-cell step.  in_* = the cell's particles (global), out_* = where the
// result goes (may alias in_*).  kLoad: copy in_* into B's arrays first;
// otherwise B.v* already hold the cell (staged in shared memory by a gather,
// or aliasing global memory).  kStore: write B.v* to out_* at the end.
template <typename Real, bool kLoad, bool kStore, class Team>
__device__ int process_cell(Team &T, const StepParams &P, CellBuf<Real> &B, CellShared &sh, const Real *in_x,
                            const Real *in_y, const Real *in_z, Real *out_x, Real *out_y, Real *out_z,
                            int n, uint32_t gcell, int32_t *m_state, double *stats_row,
                            trmcr_coll_rec *log, unsigned long long *log_count, int64_t log_cap) {
  const int tid = T.tid();
  if (n > B.n_cap) return kOverflow;
  PHASE_MARK(t_ph);
  const RngKey K{P.k0, P.k1, gcell, P.step};
  const int m0 = P.adaptive ? *m_state : P.m_fixed;
  if (n == 0) {
    if (tid == 0 && stats_row) {
      for (int k = 0; k < TRMCR_NSTATS; ++k) stats_row[k] = 0.0;
      stats_row[TRMCR_ST_MUSED] = m0;
      stats_row[TRMCR_ST_MNEXT] = m0;
    }
    return kOk;
  }
  // ---- A3: moments ----
  double s3[3] = {0, 0, 0};
  for (int i = tid; i < n; i += T.size()) {
    Real x, y, z;
    if (kLoad) load3(in_x, in_y, in_z, i, x, y, z);
    else { x = B.vx[i]; y = B.vy[i]; z = B.vz[i]; }
    if (kLoad) { B.vx[i] = x; B.vy[i] = y; B.vz[i] = z; }
    s3[0] += x; s3[1] += y; s3[2] += z;
  }
  T.template sum<3>(s3, B.red);
  const double ux = s3[0] / n, uy = s3[1] / n, uz = s3[2] / n;
  double c3[3] = {0, 0, 0};  // Pxx sum, M4 sum, centred energy
  double dv2 = 0.0;
  for (int i = tid; i < n; i += T.size()) {
    const double x = B.vx[i], y = B.vy[i], z = B.vz[i];
    const double dx = x - ux, dy = y - uy, dz = z - uz;
    const double r2 = sq3(dx, dy, dz);         // the oracle's rounding (Sigma' ties |q|)
    dv2 = fmax(dv2, r2);
    c3[0] += dx * dx;
    const double v2 = x * x + y * y + z * z;
    c3[1] += v2 * v2;
    c3[2] += r2;
  }
  for (int d = tid; d < kSplitPre; d += T.size()) {   // split uniforms, in parallel
    const uint4 w = K(kSplit, 0, (uint32_t)d, 0);
    sh.usplit[d] = u53(w.x, w.y);
  }
  T.template sum<3>(c3, B.red);
  dv2 = T.max(dv2, B.red);
  if (tid == 0) {
    sh.n = n; sh.ux = ux; sh.uy = uy; sh.uz = uz;
    sh.sums[0] = s3[0]; sh.sums[1] = s3[1]; sh.sums[2] = s3[2];
    sh.sums[3] = c3[2] + n * (ux * ux + uy * uy + uz * uz);   // sum |v|^2
    sh.S0 = (P.indicator == TRMCR_IND_PXX ? c3[0] : c3[1]) / n;
    const double rho_c = P.shock ? n * P.w_over_dx : 1.0;
    if (P.model == TRMCR_HARD_SPHERE) {
      sh.sigma = 2.0 * sqrt(dv2);            // Sigma' = 2 dv  [R4]
      sh.mu = rho_c * sh.sigma;              // mu = 4 pi rho Sigma  [R5]
    } else if (P.model == TRMCR_VHS) {
      sh.sigma = vhs_majorant(dv2, P.alpha); // Sigma' = sigma(2 dv) / K
      sh.mu = rho_c * sh.sigma;
    } else {
      sh.sigma = 0.0;
      sh.mu = rho_c;
    }
    sh.sig_run = sh.sigma;
    const double x = sh.mu * P.dt / P.eps;
    sh.p = exp(-x);
    sh.m = m0; sh.m_cur = m0; sh.flag = kOk;
    sh.prop = 0; sh.acc = 0; sh.viol = 0;
    // ---- A4: split (Alg 4.2) ----
    const int64_t N0 = ir_split(K, 0, sh.p * (double)n, sh.usplit);
    B.Q[0] = (int32_t)N0;
    sh.rem = n - N0;
    sh.d = 0;
    split_extend(K, sh, m0, B.Q, B.L_cap);
    // quotas above L_cap are zero (else split_extend flagged overflow)
    sh.r = 0; sh.lo = 1; sh.hi = sh.d < B.L_cap ? sh.d : B.L_cap;
    sh.budget = n; sh.leaf_off = 0; sh.ktot = 0; sh.nwb = 0;
  }
  T.sync();
  PHASE_ADD(0, t_ph);   // moments + split
  if (sh.flag != kOk) return sh.flag;
  Perm pi0;
  pi0.init(K(kPerm, 0, 0, 0), (uint32_t)n);
  // ---- A5/A6: attempt 0 ----
  plan_counts<Real>(T, K, B, sh);
  PHASE_ADD(1, t_ph);   // plan counts
  if (sh.flag != kOk) return sh.flag;
  plan_execute<Real>(T, P, K, B, sh, pi0, (Real)sh.sig_run, log, log_count, log_cap);
  PHASE_ADD(2, t_ph);   // plan execute
  if (tid == 0) {
    sh.Ltot = sh.L;
    sh.U = B.Q[0] < n - sh.Ltot ? B.Q[0] : n - sh.Ltot;
    sh.nT = n - sh.Ltot - sh.U;
    sh.m_next = sh.m_cur;
    sh.S_est = sh.S0; sh.E1 = 0.0;
  }
  T.sync();
  // ---- A7: TRMC-RAD ----
  if (P.adaptive) {
    for (;;) {
      rad_estimate<Real>(T, P, B, sh, pi0);
      PHASE_ADD(3, t_ph);   // RAD estimate
      if (tid == 0) {
        sh.done = 1;
        if (sh.E1 > P.delta2 && sh.m_cur < P.m_cap) {
          const int m_new = 2 * sh.m_cur < P.m_cap ? 2 * sh.m_cur : P.m_cap;
          split_extend(K, sh, m_new, B.Q, B.L_cap);
          sh.r += 1;
          sh.lo = sh.m_cur + 1;
          sh.hi = sh.d < B.L_cap ? sh.d : B.L_cap;
          sh.budget = sh.nT;
          sh.leaf_off = sh.Ltot;
          sh.m_cur = m_new;
          sh.done = 0;
        }
      }
      T.sync();
      if (sh.flag != kOk) return sh.flag;
      if (sh.done) break;
      plan_counts<Real>(T, K, B, sh);
      if (sh.flag != kOk) return sh.flag;
      plan_execute<Real>(T, P, K, B, sh, pi0, (Real)sh.sig_run, log, log_count, log_cap);
      PHASE_ADD(4, t_ph);   // RAD retries
      if (tid == 0) { sh.Ltot += sh.L; sh.nT -= sh.L; }
      T.sync();
      if (P.debug_stop > 0 && sh.r >= P.debug_stop) {
        if (kStore)
          for (int i = tid; i < n; i += T.size()) { out_x[i] = B.vx[i]; out_y[i] = B.vy[i]; out_z[i] = B.vz[i]; }
        return kOk;
      }
    }
    if (tid == 0) {
      sh.m_next = (sh.E1 < P.delta1) ? (sh.m_cur / 2 > 1 ? sh.m_cur / 2 : 1) : sh.m_cur;
    }
    T.sync();
  }
  if (P.debug_stop < 0) {   // debug: stop before the Maxwellian
    if (kStore)
      for (int i = tid; i < n; i += T.size()) { out_x[i] = B.vx[i]; out_y[i] = B.vy[i]; out_z[i] = B.vz[i]; }
    return kOk;
  }
  // ---- A8: Maxwellian of Theta ----
  PHASE_ADD(5, t_ph);
  maxwellian<Real>(T, P, K, B, sh, pi0, c3[2]);
  PHASE_ADD(6, t_ph);   // Maxwellian
  // ---- write back + stats ----
  if (kStore) {
    for (int i = tid; i < n; i += T.size()) {
      out_x[i] = B.vx[i]; out_y[i] = B.vy[i]; out_z[i] = B.vz[i];
    }
  }
  PHASE_ADD(7, t_ph);   // store
  if (tid == 0) {
    if (P.adaptive) *m_state = sh.m_next;
    if (stats_row) {
      double *s = stats_row;
      s[TRMCR_ST_N] = n; s[TRMCR_ST_P] = sh.p; s[TRMCR_ST_MU] = sh.mu; s[TRMCR_ST_SIGMA] = sh.sigma;
      s[TRMCR_ST_S0] = sh.S0; s[TRMCR_ST_SEST] = sh.S_est; s[TRMCR_ST_E1] = sh.E1;
      s[TRMCR_ST_MUSED] = sh.m_cur; s[TRMCR_ST_MNEXT] = sh.m_next; s[TRMCR_ST_DEPTH] = sh.d;
      s[TRMCR_ST_ATTEMPTS] = sh.r + 1; s[TRMCR_ST_LEAVES] = sh.Ltot; s[TRMCR_ST_UNTOUCHED] = sh.U;
      s[TRMCR_ST_THERMALISED] = sh.nT; s[TRMCR_ST_PROPOSALS] = (double)sh.prop;
      s[TRMCR_ST_ACCEPTED] = (double)sh.acc; s[TRMCR_ST_VIOLATIONS] = (double)sh.viol;
      s[TRMCR_ST_MAXW] = sh.nT + sh.nwb >= 2 ? sh.nT + sh.nwb : 0;
      s[TRMCR_ST_PX] = sh.sums[0]; s[TRMCR_ST_PY] = sh.sums[1]; s[TRMCR_ST_PZ] = sh.sums[2];
      s[TRMCR_ST_ENERGY] = sh.sums[3];
    }
  }
  return kOk;
}

}  // namespace trmcr
