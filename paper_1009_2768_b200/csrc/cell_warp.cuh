// cell_warp.cuh — the general collision step (A3-A8, trees included) with one
// WARP per cell: the same computation as process_cell (cell_step.cuh, one CTA
// per cell) and the same keyed draws, but every phase is warp-synchronous
// (__syncwarp only, no CTA barrier), so a CTA of 8 warps advances 8 cells
// independently.  Each warp owns a shared-memory slab (velocities + plan).
// A cell larger than the slab, or whose tree outgrows it, is left untouched
// and queued for the CTA kernel (which in turn queues giants for the
// global-memory kernel).
#pragma once
#include "cell_step.cuh"
#include <type_traits>

namespace trmcr {

constexpr int kWarpCellWarps = 4;
constexpr int kWarpSplitPre = 32;      // split uniforms drawn up front: one per lane (deeper levels draw theirs)
#ifndef TRMCR_WARP_MINB
#define TRMCR_WARP_MINB 4        // CTAs of kWarpCellWarps warps per SM the register budget allows (128 regs)
#endif

// fp32 moment passes over the n particles (vx, vy, vz)[0..n) of a cell, with
// the warp.  The sums are defined on the particle INDEX only: class k (0..127)
// is the sequential fp32 sum of particles k, k + 128, k + 256, ...; lane L's
// partial is (class 4L + class 4L+1) + (class 4L+2 + class 4L+3); the warp sum
// (fp64) of the lane partials follows.  So the mean, Sigma', p and everything
// derived from them do not depend on where the cell lies in the array (single
// domain or slab: bitwise).  The loads, though, are always 16-byte ones: a
// cell whose first particle sits k elements past a 16-byte boundary is read
// from that boundary, so lane L's four accumulators hold classes 4L - k .. 4L
// - k + 3 (mod 128; the slots before particle 0 and after particle n - 1 are
// skipped), each still summed in index order; warp_cell_fold puts the classes
// back with three shuffles.  Four independent add chains per lane and sum.
// f(slot<J>, x, y, z) adds particle (x, y, z) to accumulator J of each sum.
#ifndef TRMCR_SUMS_UNROLL
#define TRMCR_SUMS_UNROLL 4      // 16-byte groups per lane in flight in the first pass over a cell (load latency)
#endif
#ifndef TRMCR_CENTRAL_UNROLL
#define TRMCR_CENTRAL_UNROLL 2
#endif
template <int J> using slot = std::integral_constant<int, J>;
__device__ __forceinline__ uint32_t misalign4(const float *p) {
  return (((uint32_t)reinterpret_cast<uintptr_t>(p)) >> 2) & 3u;
}
template <int U, typename F>
__device__ __forceinline__ uint32_t warp_cell_for4(const float *vx, const float *vy, const float *vz, int n, F &&f) {
  const int lane = threadIdx.x & 31;
  const int k = (int)misalign4(vx);
  if ((uint32_t)k != misalign4(vy) || (uint32_t)k != misalign4(vz)) __trap();   // the three arrays are shifted alike (capacities are multiples of 4)
  const float4 *X = reinterpret_cast<const float4 *>(vx - k), *Y = reinterpret_cast<const float4 *>(vy - k),
               *Z = reinterpret_cast<const float4 *>(vz - k);
  // 16-byte groups q = 0 .. nv-1; group q holds particles 4q - k .. 4q - k + 3.  Those wholly
  // inside the cell are [k > 0, q1); group 0 (k > 0) and group q1 (if (n + k) % 4) are partial.
  const int q1 = (n + k) >> 2, nv = (n + k + 3) >> 2;
  auto edge = [&](int q) {       // slots outside [0, n) belong to the neighbouring cells
    const float4 a = X[q], b = Y[q], c = Z[q];
    const int lo = 4 * q - k;
    if ((unsigned)lo < (unsigned)n) f(slot<0>{}, a.x, b.x, c.x);
    if ((unsigned)(lo + 1) < (unsigned)n) f(slot<1>{}, a.y, b.y, c.y);
    if ((unsigned)(lo + 2) < (unsigned)n) f(slot<2>{}, a.z, b.z, c.z);
    if ((unsigned)(lo + 3) < (unsigned)n) f(slot<3>{}, a.w, b.w, c.w);
  };
  const bool head = k > 0 && lane == 0, tail = nv > q1 && (q1 & 31) == lane && !(k > 0 && q1 == 0);
  if (head) edge(0);             // first in lane 0's order
#pragma unroll U
  for (int q = head ? 32 : lane; q < q1; q += 32) {
    const float4 a = X[q], b = Y[q], c = Z[q];
    f(slot<0>{}, a.x, b.x, c.x); f(slot<1>{}, a.y, b.y, c.y); f(slot<2>{}, a.z, b.z, c.z); f(slot<3>{}, a.w, b.w, c.w);
  }
  if (tail) edge(q1);            // last in its lane's order
  return (uint32_t)k;
}
// Lane partial of one sum from its four accumulators (k = warp_cell_for4's result; whole warp).
__device__ __forceinline__ float warp_cell_fold(const float (&a)[4], uint32_t k) {
  const int nxt = ((threadIdx.x & 31) + 1) & 31;
  const float t0 = __shfl_sync(0xffffffffu, a[0], nxt), t1 = __shfl_sync(0xffffffffu, a[1], nxt),
              t2 = __shfl_sync(0xffffffffu, a[2], nxt);
  const float c0 = k == 0 ? a[0] : k == 1 ? a[1] : k == 2 ? a[2] : a[3];
  const float c1 = k == 0 ? a[1] : k == 1 ? a[2] : k == 2 ? a[3] : t0;
  const float c2 = k == 0 ? a[2] : k == 1 ? a[3] : k == 2 ? t0 : t1;
  const float c3 = k == 0 ? a[3] : k == 1 ? t0 : k == 2 ? t1 : t2;
  return (c0 + c1) + (c2 + c3);
}
// Pass 1: lane partials of sum v (to be warp-summed in fp64).
__device__ __forceinline__ void warp_cell_sums(const float *vx, const float *vy, const float *vz, int n, double &sx,
                                               double &sy, double &sz) {
  float ax[4] = {0, 0, 0, 0}, ay[4] = {0, 0, 0, 0}, az[4] = {0, 0, 0, 0};
  const uint32_t k = warp_cell_for4<TRMCR_SUMS_UNROLL>(vx, vy, vz, n, [&](auto J, float x, float y, float z) {
    constexpr int j = decltype(J)::value;
    ax[j] += x; ay[j] += y; az[j] += z;
  });
  sx = warp_cell_fold(ax, k); sy = warp_cell_fold(ay, k); sz = warp_cell_fold(az, k);
}
// Pass 2: lane partials of sum (v_x - u_x)^2, sum |v|^4, sum |v - u|^2 and the lane's max |v - u|^2.
__device__ __forceinline__ void warp_cell_central(const float *vx, const float *vy, const float *vz, int n, float fux,
                                                  float fuy, float fuz, double &c0, double &c1, double &c2,
                                                  double &dv2) {
  float f0[4] = {0, 0, 0, 0}, f1[4] = {0, 0, 0, 0}, f2[4] = {0, 0, 0, 0}, fm = 0;
  const uint32_t k = warp_cell_for4<TRMCR_CENTRAL_UNROLL>(vx, vy, vz, n, [&](auto J, float x, float y, float z) {
    // explicit roundings: the loop body and the edge groups are separate inlined copies and
    // must not be contracted differently (a particle's copy depends on the cell's alignment)
    const float dx = __fsub_rn(x, fux), dy = __fsub_rn(y, fuy), dz = __fsub_rn(z, fuz);
    const float xx = __fmul_rn(dx, dx);
    const float r2 = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, xx));
    fm = fmaxf(fm, r2);
    constexpr int j = decltype(J)::value;
    f0[j] = __fadd_rn(f0[j], xx);
    const float v2 = __fmaf_rn(z, z, __fmaf_rn(y, y, __fmul_rn(x, x)));
    f1[j] = __fmaf_rn(v2, v2, f1[j]);
    f2[j] = __fadd_rn(f2[j], r2);
  });
  c0 = warp_cell_fold(f0, k); c1 = warp_cell_fold(f1, k); c2 = warp_cell_fold(f2, k); dv2 = fm;
}

// Generic visit of a cell with the warp (the A9 moments kernel, fp64 sums): f(i, x, y, z)
// per particle; round r gives lane L particles 4 (32 r + L) .. + 3 (index only),
// 16-byte loads when the cell is 16-byte aligned; fp64 cells lane-strided.
template <typename Real, typename F>
__device__ __forceinline__ void warp_cell_fori(const Real *vx, const Real *vy, const Real *vz, int n, F &&f) {
  const int lane = threadIdx.x & 31;
  if constexpr (sizeof(Real) == 4) {
    const int body = n >> 2;
    const bool al = (((uint32_t)reinterpret_cast<uintptr_t>(vx)) & 15u) == 0u;
    for (int q = lane; q < body; q += 32) {
      const int i = 4 * q;
      float4 a, b, c;
      if (al) {
        a = *reinterpret_cast<const float4 *>(vx + i);
        b = *reinterpret_cast<const float4 *>(vy + i);
        c = *reinterpret_cast<const float4 *>(vz + i);
      } else {
        a = make_float4(vx[i], vx[i + 1], vx[i + 2], vx[i + 3]);
        b = make_float4(vy[i], vy[i + 1], vy[i + 2], vy[i + 3]);
        c = make_float4(vz[i], vz[i + 1], vz[i + 2], vz[i + 3]);
      }
      f(i, a.x, b.x, c.x); f(i + 1, a.y, b.y, c.y); f(i + 2, a.z, b.z, c.z); f(i + 3, a.w, b.w, c.w);
    }
    const int t = 4 * body + lane;
    if (t < n) f(t, vx[t], vy[t], vz[t]);
  } else {
    for (int i = lane; i < n; i += 32) f(i, vx[i], vy[i], vz[i]);
  }
}
// (the same without the slot index)
template <typename Real, typename F>
__device__ __forceinline__ void warp_cell_for(const Real *vx, const Real *vy, const Real *vz, int n, F &&f) {
  warp_cell_fori<Real>(vx, vy, vz, n, [&](int, Real x, Real y, Real z) { f(x, y, z); });
}

// Per-warp scalars (in the warp's slab, lane 0 writes, __syncwarp publishes).
struct WarpShared {
  double ux, uy, uz, S0, sigma, p, mu, S_est, E1, c2;
  double cind, dS;            // pre-step indicator sum (n S0) and its change by the collisions so far
  double sig_run;             // running majorant (sigma_update) [R33]
  uint4 pk;                // key of pi0
  PermDom D0;              // its domain [0, n)
  double sums[4];
  int n, m_cur, m_next, d, top, lo, hi, r, flag, done;
  int64_t rem;
  int32_t L, Ltot, U, nT, budget, leaf_off, ktot, nwb;
  unsigned long long prop, acc, viol;
};


struct WarpSlabLayout {
  int n_cap, K_cap, L_cap, v_smem;   // v_smem = 0: the cell's velocities live in global memory
  size_t per_warp;   // bytes of one warp's slab incl. WarpShared (16-byte multiple)
  int wb;
  size_t off_v, off_ctype, off_crank, off_cslot, off_ints, off_rk, off_pdom, off_u, off_red, off_sh, off_wlen,
      off_wused;
  void build(int n, int K, int L, size_t rs, int v_in_smem, int wb_on = 0) {
    n_cap = n; K_cap = K; L_cap = L; v_smem = v_in_smem; wb = wb_on;
    size_t o = 0;
    auto al = [&](size_t a) { o = (o + a - 1) / a * a; };
    off_red = o; o += 8 * sizeof(double);
    al(16); off_rk = o; o += (size_t)(L + 1) * sizeof(uint4);
    off_pdom = o; o += (size_t)(L + 1) * sizeof(PermDom);
    off_u = o; o += (size_t)kWarpSplitPre * sizeof(double);
    al(16); off_v = o; if (v_in_smem) o += 3 * (size_t)n * rs;
    al(16); off_cslot = o; o += (size_t)K * 4;     // 2 K uint16
    off_crank = o; o += (size_t)K * 2;             // K uint16
    off_ctype = o; o += (size_t)K;                 // K uint8
    off_ints = o; o += 6 * (size_t)(L + 1) * 4;
    al(16); off_wlen = o; if (wb) o += (size_t)K * 8;
    off_wused = o; if (wb) o += (size_t)K * 2;
    al(16); off_sh = o; o += sizeof(WarpShared);
    al(16); per_warp = o;
  }
};

template <typename Real>
__device__ __forceinline__ void bind_warp_slab(CellBuf<Real> &B, unsigned char *base, const WarpSlabLayout &Lay,
                                               double *&usplit) {
  B.red = reinterpret_cast<double *>(base + Lay.off_red);
  B.rk = reinterpret_cast<uint4 *>(base + Lay.off_rk);
  usplit = reinterpret_cast<double *>(base + Lay.off_u);
  Real *v = reinterpret_cast<Real *>(base + Lay.off_v);
  B.vx = v; B.vy = v + Lay.n_cap; B.vz = v + 2 * Lay.n_cap;   // rebound per cell when !v_smem
  B.ctype = nullptr; B.crank = nullptr; B.cslot = nullptr;
  B.ctype8 = reinterpret_cast<uint8_t *>(base + Lay.off_ctype);
  B.crank16 = reinterpret_cast<uint16_t *>(base + Lay.off_crank);
  B.cslot16 = reinterpret_cast<uint16_t *>(base + Lay.off_cslot);
  int32_t *ints = reinterpret_cast<int32_t *>(base + Lay.off_ints);
  const int Lp = Lay.L_cap + 1;
  B.Q = ints; B.C = ints + Lp; B.S = ints + 2 * Lp; B.cons = ints + 3 * Lp;
  B.base = ints + 4 * Lp; B.cnt = ints + 5 * Lp;
  B.pdom = reinterpret_cast<PermDom *>(base + Lay.off_pdom);
  B.wlen = Lay.wb ? reinterpret_cast<double *>(base + Lay.off_wlen) : nullptr;
  B.wused = Lay.wb ? reinterpret_cast<uint8_t *>(base + Lay.off_wused) : nullptr;
  B.mask = nullptr;
  B.n_cap = Lay.n_cap; B.K_cap = Lay.K_cap; B.L_cap = Lay.L_cap;
}

// ---- warp versions of the phases (same definitions as cell_step.cuh) ----

__device__ __forceinline__ void wsplit_extend(const RngKey &K, WarpShared &sh, int m, int32_t *Q, int L_cap,
                                              const double *usplit) {
  while (sh.rem > 0 && sh.d < m) {
    const double y = sh.p * (double)sh.rem;
    if (y < 0x1p-53) {
      for (int d = sh.d + 1; d <= m && d <= L_cap; ++d) Q[d] = 0;
      sh.d = m;
      break;
    }
    sh.d++;
    int64_t q = ir_split(K, sh.d, y, usplit, kWarpSplitPre);
    if (q > sh.rem) q = sh.rem;
    if (sh.d <= L_cap) Q[sh.d] = (int32_t)q;
    else if (q > 0) sh.flag = kOverflow;
    sh.rem -= q;
  }
}

template <typename Real>
__device__ void wplan_counts(const RngKey &K, CellBuf<Real> &B, WarpShared &sh) {
  const int lane = threadIdx.x & 31;
  int top = sh.hi;
  while (top >= sh.lo && B.Q[top] == 0) top--;
  for (;;) {
    if (top < sh.lo || top < 1) {
      __syncwarp();
      if (lane == 0) { sh.top = 0; sh.L = 0; }
      __syncwarp();
      return;
    }
    if (top > B.L_cap) {
      __syncwarp();
      if (lane == 0) sh.flag = kOverflow;
      __syncwarp();
      return;
    }
    for (int d = lane; d <= top; d += 32) B.cons[d] = 0;
    __syncwarp();
    int Sacc = 0;
    for (int d = top; d >= 1; --d) {
      const int Qd = (d >= sh.lo) ? B.Q[d] : 0;
      const int Cd = (Qd + B.cons[d] + 1) >> 1;
      if ((int64_t)Sacc + Cd > B.K_cap) {
        __syncwarp();
        if (lane == 0) sh.flag = kOverflow;
        __syncwarp();
        return;
      }
      __syncwarp();
      if (lane == 0) { B.C[d] = Cd; B.S[d] = Sacc; }
      for (int j = lane; j < Cd; j += 32) {
        const uint32_t w = K(kType, sh.r, d, j).x;
        const uint32_t a = __umulhi(w, (uint32_t)d);
        B.ctype8[Sacc + j] = (uint8_t)a;
        atomicAdd(&B.cons[a], 1);
        atomicAdd(&B.cons[d - 1 - a], 1);
      }
      Sacc += Cd;
      __syncwarp();
    }
    if (B.cons[0] <= sh.budget) {
      __syncwarp();
      if (lane == 0) { sh.L = B.cons[0]; sh.top = top; }
      __syncwarp();
      return;
    }
    int t = top - 1;                       // guard: drop the top quota level
    while (t >= sh.lo && B.Q[t] == 0) t--;
    top = t;
    __syncwarp();
  }
}

// Bottom-up slot resolution + execution (as plan_execute, cell_step.cuh) in
// three warp passes: (1) per level, the stable in-level ranks and each side's
// demand index on its pool (pool 0: the cell's leaf order), (2) ALL keyed
// permutation evaluations of the attempt in one flat pass over its 2 ktot
// demands - lanes are not left idle by small levels, two walks interleaved per
// lane - and (3) per level, pool outputs to slots and the collisions.
template <typename Real, bool WB, int MOD = -1>
__device__ void wplan_execute(const StepParams &P, const RngKey &K, CellBuf<Real> &B, WarpShared &sh,
                              const Perm &pi0, Real sigma, trmcr_coll_rec *log, unsigned long long *log_count,
                              int64_t log_cap) {
  const int lane = threadIdx.x & 31;
  const int top = sh.top;
  if (top < 1) return;
  for (int d = lane; d <= top; d += 32) {
    B.base[d] = 0;
    B.cnt[d] = 0;
    if (d >= 1) {
      B.rk[d] = K(kPerm, sh.r, d, 0);
      B.pdom[d] = perm_dom(2u * (uint32_t)B.C[d]);
    }
  }
  const int ktot = B.S[1] + B.C[1];                // collisions of the plan (levels top..1 stored from 0)
  if (WB && P.wb) for (int o = lane; o < 2 * ktot; o += 32) B.wused[o] = 0;
  if (lane == 0) sh.ktot = ktot;
  __syncwarp();
  const int r = sh.r, leaf_off = sh.leaf_off, n = sh.n;
  // ---- pass 1: demand indices (permutation inputs) into cslot16, level into crank16 ----
  int pd = 0;
  for (int d = 1; d <= top; ++d) {
    const int Cd = B.C[d], Sd = B.S[d];
    if (Cd == 0) continue;
    if (pd > 0) {                          // fold level pd into base[], clear its histogram
      for (int p = lane; p < pd; p += 32) B.cons[p] = B.base[p] + B.cnt[p] + B.cnt[pd - 1 - p];
      __syncwarp();
      for (int p = lane; p < pd; p += 32) { B.base[p] = B.cons[p]; B.cnt[p] = 0; }
      __syncwarp();
    }
    for (int j0 = 0; j0 < Cd; j0 += 32) {  // stable in-level ranks per type
      const int j = j0 + lane;
      const bool valid = j < Cd;
      const uint32_t a = valid ? (uint32_t)B.ctype8[Sd + j] : 0xFFFFFFFFu;
      const unsigned peers = __match_any_sync(0xffffffffu, a);
      const unsigned lt = (1u << lane) - 1u;
      int c0 = 0;
      if (valid) c0 = B.cnt[a];
      __syncwarp();
      if (valid) {
        B.crank16[Sd + j] = (uint16_t)(c0 + __popc(peers & lt));
        if ((peers & lt) == 0u) B.cnt[a] = c0 + __popc(peers);
      }
      __syncwarp();
    }
    pd = d;
    for (int j = lane; j < Cd; j += 32) {
      const uint32_t a = B.ctype8[Sd + j], b = (uint32_t)d - 1u - a;
      const uint32_t rank = B.crank16[Sd + j];
      const uint32_t t0 = (uint32_t)B.base[a] + rank, t1 = (uint32_t)(B.base[b] + B.cnt[b]) + rank;
      B.cslot16[2 * (Sd + j)] = (uint16_t)(a == 0 ? (uint32_t)leaf_off + t0 : t0);
      B.cslot16[2 * (Sd + j) + 1] = (uint16_t)(b == 0 ? (uint32_t)leaf_off + t1 : t1);
      B.crank16[Sd + j] = (uint16_t)d;
    }
    __syncwarp();
  }
  PHASE_MARK(t_p2);
  // ---- pass 2: every permutation of the attempt, lanes over demands ----
  for (int q0 = 0; q0 < 2 * ktot; q0 += 64) {
    uint32_t x[2], pool[2];
    bool on[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int q = q0 + 32 * h + lane;
      on[h] = q < 2 * ktot;
      x[h] = 0xFFFFFFFFu; pool[h] = 0;
      if (on[h]) {
        const int k = q >> 1;
        const uint32_t a = B.ctype8[k], d = B.crank16[k];
        pool[h] = (q & 1) ? d - 1u - a : a;
        x[h] = B.cslot16[q];
      }
    }
    uint32_t y[2];
    perm_eval2(x[0], pool[0] == 0 ? pi0.rk : B.rk[pool[0]], pool[0] == 0 ? pi0.D : B.pdom[pool[0]],
               x[1], pool[1] == 0 ? pi0.rk : B.rk[pool[1]], pool[1] == 0 ? pi0.D : B.pdom[pool[1]], y[0], y[1]);
#pragma unroll
    for (int h = 0; h < 2; ++h)
      if (on[h]) B.cslot16[q0 + 32 * h + lane] = (uint16_t)(y[h] == 0xFFFFFFFFu ? 0xFFFFu : y[h]);
  }
  __syncwarp();
  WPHASE_ADD(12, t_p2);   // plan_execute pass 2 (permutations)
  // ---- pass 3: slots and collisions, level by level ----
  unsigned acc = 0, viol = 0;
  unsigned long long prop = 0;
  double dS = 0.0;                         // this lane's share of the indicator change (RAD)
  double *dSp = P.adaptive ? &dS : nullptr;
  const Real iux = (Real)sh.ux;
  for (int d = 1; d <= top; ++d) {
    const int Cd = B.C[d], Sd = B.S[d];
    if (Cd == 0) continue;
    for (int j = lane; j < Cd; j += 32) {
      const uint32_t a = B.ctype8[Sd + j], b = (uint32_t)d - 1u - a;
      const uint32_t pool[2] = {a, b};
      uint32_t slot[2], y[2];
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        y[s] = B.cslot16[2 * (Sd + j) + s];
        slot[s] = (pool[s] == 0 || y[s] == 0xFFFFu) ? y[s] : (uint32_t)B.cslot16[2u * (uint32_t)B.S[pool[s]] + y[s]];
        if (slot[s] >= (uint32_t)n) { atomicOr(P.err, kErrInternal); slot[s] = 0; }
      }
      if (WB && P.wb) {                      // TRMC-WB: lengths, consumed outputs
        double ln[2] = {0.0, 0.0};
#pragma unroll
        for (int s = 0; s < 2; ++s)
          if (pool[s] != 0 && y[s] != 0xFFFFu) {
            const uint32_t o = 2u * (uint32_t)B.S[pool[s]] + y[s];
            B.wused[o] = 1;
            ln[s] = B.wlen[o >> 1];
          }
        B.wlen[Sd + j] = wb_combine(P.wb, d, ln[0], ln[1]);
      }
      B.cslot16[2 * (Sd + j)] = (uint16_t)slot[0];
      B.cslot16[2 * (Sd + j) + 1] = (uint16_t)slot[1];
      if (!(WB && P.sigma_update)) {
        const int ok = tree_collision<Real, MOD>(P, K, B, sigma, r, d, (uint32_t)j, slot[0], slot[1], viol, dSp, iux);
        acc += ok;
        log_collision(P, K, log, log_count, log_cap, r, d, j, ok, slot[0], slot[1]);
      }
    }
    if (WB && P.sigma_update) {              // majorant raised after each proposal [R33]
      __syncwarp();
      double mx = 0.0;
      for (int j = lane; j < Cd; j += 32)
        mx = fmax(mx, (double)pair_sigma<Real>(P, B, B.cslot16[2 * (Sd + j)], B.cslot16[2 * (Sd + j) + 1]));
      mx = warp_max(mx);
      if (mx > (double)viol_bound(sigma)) {  // a violation in this level: canonical order, one lane
        if (lane == 0)
          for (int j = 0; j < Cd; ++j) {
            const uint32_t s0 = B.cslot16[2 * (Sd + j)], s1 = B.cslot16[2 * (Sd + j) + 1];
            const Real sj = pair_sigma<Real>(P, B, s0, s1);
            const int ok = tree_collision<Real, MOD>(P, K, B, sigma, r, d, (uint32_t)j, s0, s1, viol, dSp, iux);
            acc += ok;
            log_collision(P, K, log, log_count, log_cap, r, d, j, ok, s0, s1);
            if (sj > viol_bound(sigma)) sigma = sj;
          }
        sigma = __shfl_sync(0xffffffffu, sigma, 0);
      } else {
        for (int j = lane; j < Cd; j += 32) {
          const uint32_t s0 = B.cslot16[2 * (Sd + j)], s1 = B.cslot16[2 * (Sd + j) + 1];
          const int ok = tree_collision<Real, MOD>(P, K, B, sigma, r, d, (uint32_t)j, s0, s1, viol, dSp, iux);
          acc += ok;
          log_collision(P, K, log, log_count, log_cap, r, d, j, ok, s0, s1);
        }
      }
    }
    prop += (unsigned long long)Cd;
    __syncwarp();
  }
  WPHASE_ADD(13, t_p2);   // plan_execute pass 3 (collisions)
  if (WB && P.sigma_update && lane == 0) sh.sig_run = (double)sigma;
  acc = __reduce_add_sync(0xffffffffu, acc);
  viol = __reduce_add_sync(0xffffffffu, viol);
  if (P.adaptive) dS = warp_sum_call(dS);
  if (lane == 0) { sh.prop += prop; sh.acc += acc; sh.viol += viol; sh.dS += dS; }
  __syncwarp();
}

// RAD indicator estimate with Theta taken analytically, as
// rad_estimate (cell_step.cuh) but without a pass over the whole cell: the sum
// of the indicator over all slots is its pre-step value plus the change the
// collisions made (accumulated in pass 3), so only Theta's slots are read.
template <typename Real>
__device__ void wrad_estimate(const StepParams &P, CellBuf<Real> &B, WarpShared &sh, const Perm &pi0) {
  const int lane = threadIdx.x & 31, n = sh.n, nT = sh.nT;
  const bool pxx = P.indicator == TRMCR_IND_PXX;
  const double ux = sh.ux;
  double v1 = 0, tx = 0, ty = 0, tz = 0, t2 = 0;
  for (int q = lane; q < nT; q += 32) {
    const uint32_t s = pi0((uint32_t)(sh.Ltot + q));
    if (s >= (uint32_t)n) { atomicOr(P.err, kErrInternal); continue; }
    const double x = B.vx[s], y = B.vy[s], z = B.vz[s];
    if (pxx) { const double dx = x - ux; v1 += dx * dx; }
    else { const double v2 = x * x + y * y + z * z; v1 += v2 * v2; }
    tx += x; ty += y; tz += z; t2 += x * x + y * y + z * z;
  }
  if (__any_sync(0xffffffffu, nT > 0)) {
    v1 = warp_sum_call(v1); tx = warp_sum_call(tx); ty = warp_sum_call(ty); tz = warp_sum_call(tz);
    t2 = warp_sum_call(t2);
  }
  if (lane == 0) {
    double s = (sh.cind + sh.dS) - v1;
    if (nT > 0) {
      tx /= nT; ty /= nT; tz /= nT;
      const double T = fmax(0.0, t2 / nT - (tx * tx + ty * ty + tz * tz)) / 3.0;
      if (pxx) {
        s += (double)nT * (T + (tx - ux) * (tx - ux));
      } else {
        const double u2 = tx * tx + ty * ty + tz * tz;
        s += (double)nT * (u2 * u2 + 10.0 * u2 * T + 15.0 * T * T);
      }
    }
    sh.S_est = s / n;
    sh.E1 = sh.S0 != 0.0 ? fabs(sh.S_est - sh.S0) / fabs(sh.S0) : (sh.S_est == 0.0 ? 0.0 : INFINITY);
  }
  __syncwarp();
}

// Conservative Maxwellian (A8) over Theta = pi0 positions [Ltot, Ltot + nT)
// plus, under TRMC-WB, the final outputs whose tree is longer than wb_max:
// index q < nT is pi0(Ltot + q); q >= nT is output q - nT of the plan.
template <typename Real, bool WB>
__device__ void wmaxwellian(const StepParams &P, const RngKey &K, CellBuf<Real> &B, WarpShared &sh,
                            const Perm &pi0, double ec_all) {
  const int lane = threadIdx.x & 31, nT = sh.nT;
  const int nq = nT + ((WB && P.wb) ? 2 * sh.ktot : 0);
  auto member = [&](int q, uint32_t &s) -> bool {
    if (!WB || q < nT) { s = pi0((uint32_t)(sh.Ltot + q)); return true; }
    const int o = q - nT;
    if (B.wused[o] || !(B.wlen[o >> 1] > (double)P.wb_max)) return false;
    s = B.cslot16[o];
    return true;
  };
  int nwb = 0;
  if (WB && P.wb) {
    for (int o = lane; o < 2 * sh.ktot; o += 32) nwb += (!B.wused[o] && B.wlen[o >> 1] > (double)P.wb_max) ? 1 : 0;
    nwb = __reduce_add_sync(0xffffffffu, nwb);
  }
  if (lane == 0) sh.nwb = nwb;
  const int nTT = nT + nwb;
  if (nTT < 2) return;
  const bool full = (nT == sh.n);
  double ux, uy, uz;
  if (full) {
    ux = sh.ux; uy = sh.uy; uz = sh.uz;
  } else {
    double a = 0, b = 0, c = 0;
    for (int q = lane; q < nq; q += 32) {
      uint32_t s;
      if (!member(q, s)) continue;
      if (s >= (uint32_t)sh.n) { atomicOr(P.err, kErrInternal); continue; }
      a += (double)B.vx[s]; b += (double)B.vy[s]; c += (double)B.vz[s];
    }
    ux = warp_sum_call(a) / nTT; uy = warp_sum_call(b) / nTT; uz = warp_sum_call(c) / nTT;
  }
  double g0s = 0, g1s = 0, g2s = 0, gg = 0, ec = 0;
  for (int q = lane; q < nq; q += 32) {
    uint32_t s = (uint32_t)q;
    if (!full && !member(q, s)) continue;
    if (s >= (uint32_t)sh.n) continue;
    if (!full) {
      const double dx = B.vx[s] - ux, dy = B.vy[s] - uy, dz = B.vz[s] - uz;
      ec += dx * dx + dy * dy + dz * dz;
    }
    Real g0, g1, g2;
    gauss3<Real>(K, s, g0, g1, g2);
    B.vx[s] = g0; B.vy[s] = g1; B.vz[s] = g2;
    g0s += g0; g1s += g1; g2s += g2;
    gg += (double)g0 * g0 + (double)g1 * g1 + (double)g2 * g2;
  }
  g0s = warp_sum_call(g0s); g1s = warp_sum_call(g1s); g2s = warp_sum_call(g2s); gg = warp_sum_call(gg);
  ec = full ? ec_all : warp_sum_call(ec);
  const double gx = g0s / nTT, gy = g1s / nTT, gz = g2s / nTT;
  const double D = gg - nTT * (gx * gx + gy * gy + gz * gz);
  const double sc = (D > 0.0 && ec > 0.0) ? sqrt(ec / D) : 0.0;
  const Real rsc = (Real)sc, rgx = (Real)gx, rgy = (Real)gy, rgz = (Real)gz;
  const Real rux = (Real)ux, ruy = (Real)uy, ruz = (Real)uz;
  __syncwarp();
  for (int q = lane; q < nq; q += 32) {
    uint32_t s = (uint32_t)q;
    if (!full && !member(q, s)) continue;
    if (s >= (uint32_t)sh.n) continue;
    B.vx[s] = rux + rsc * (B.vx[s] - rgx);
    B.vy[s] = ruy + rsc * (B.vy[s] - rgy);
    B.vz[s] = ruz + rsc * (B.vz[s] - rgz);
  }
  __syncwarp();
}

// WB: compile the TRMC-WB bookkeeping in (the kernels are instantiated with and
// without it; the hot path without carries no extra code or registers).
// The general step of one cell in three phases that communicate through the
// warp's WarpShared (so a CTA can run its warps' cells phase by phase in lock
// step, keeping one phase's code in the instruction cache):
//   wphase_begin    A3 moments, A4 split, pi0 key
//   wphase_attempt  A5/A6 plan + collisions of one attempt, then A7's estimate
//                   and decision (sh.done = 1 when no retry follows)
//   wphase_end      A8 Maxwellian, m_state, statistics row
// Each returns kOk or an overflow flag (the cell is then left for the CTA path).
template <typename Real, int MOD = -1>
__device__ int wphase_begin(const StepParams &P, CellBuf<Real> &B, WarpShared &sh, double *usplit, double sx,
                            double sy, double sz, int n, uint32_t gcell, const int32_t *m_state) {
  const int lane = threadIdx.x & 31;
  const RngKey K{P.k0, P.k1, gcell, P.step};
  const int m0 = P.adaptive ? *m_state : P.m_fixed;
  // ---- A3: moments ----
  const double Sx = warp_sum_call(sx), Sy = warp_sum_call(sy), Sz = warp_sum_call(sz);
  const double ux = Sx / n, uy = Sy / n, uz = Sz / n;
  double c0 = 0, c1 = 0, c2 = 0, dv2 = 0;
  if constexpr (sizeof(Real) == 4) {
    // fp32 statistical mode: fp32 lane partials (~n/32 terms), fp64 warp sums
    const float fux = (float)ux, fuy = (float)uy, fuz = (float)uz;
    warp_cell_central(B.vx, B.vy, B.vz, n, fux, fuy, fuz, c0, c1, c2, dv2);
  } else {
    for (int i = lane; i < n; i += 32) {
      const double x = B.vx[i], y = B.vy[i], z = B.vz[i];
      const double dx = x - ux, dy = y - uy, dz = z - uz;
      const double r2 = sq3(dx, dy, dz);       // the oracle's rounding (Sigma' ties |q|)
      dv2 = fmax(dv2, r2);
      c0 += dx * dx;
      const double v2 = x * x + y * y + z * z;
      c1 += v2 * v2;
      c2 += r2;
    }
  }
  {                                              // split uniforms of levels < 32, one per lane
    const uint4 w = K(kSplit, 0, (uint32_t)lane, 0);
    usplit[lane] = u53(w.x, w.y);
  }
  const uint4 pk = K(kPerm, 0, 0, 0);
  c0 = warp_sum_call(c0); c1 = warp_sum_call(c1); c2 = warp_sum_call(c2); dv2 = warp_max_call(dv2);
  __syncwarp();
  if (lane == 0) {
    sh.n = n; sh.ux = ux; sh.uy = uy; sh.uz = uz; sh.c2 = c2; sh.pk = pk; sh.D0 = perm_dom((uint32_t)n);
    sh.sums[0] = Sx; sh.sums[1] = Sy; sh.sums[2] = Sz; sh.sums[3] = c2 + n * (ux * ux + uy * uy + uz * uz);
    sh.cind = P.indicator == TRMCR_IND_PXX ? c0 : c1;
    sh.dS = 0.0;
    sh.S0 = sh.cind / n;
    const double rho_c = P.shock ? n * P.w_over_dx : 1.0;
    const int model = MOD >= 0 ? MOD : P.model;
    if (model == TRMCR_HARD_SPHERE) { sh.sigma = 2.0 * sqrt(dv2); sh.mu = rho_c * sh.sigma; }
    else if (model == TRMCR_VHS) { sh.sigma = vhs_majorant(dv2, P.alpha); sh.mu = rho_c * sh.sigma; }
    else { sh.sigma = 0.0; sh.mu = rho_c; }
    sh.sig_run = sh.sigma;
    sh.p = exp(-(sh.mu * P.dt / P.eps));
    sh.m_cur = m0; sh.flag = kOk;
    sh.prop = 0; sh.acc = 0; sh.viol = 0;
    // ---- A4: split ----
    const int64_t N0 = ir_split(K, 0, sh.p * (double)n, usplit, kWarpSplitPre);
    B.Q[0] = (int32_t)N0;
    sh.rem = n - N0;
    sh.d = 0;
    wsplit_extend(K, sh, m0, B.Q, B.L_cap, usplit);
    sh.r = 0; sh.lo = 1; sh.hi = sh.d < B.L_cap ? sh.d : B.L_cap;
    sh.budget = n; sh.leaf_off = 0;
    sh.done = 0; sh.ktot = 0; sh.nwb = 0;
  }
  __syncwarp();
  return sh.flag;
}

template <typename Real, bool WB, int MOD = -1>
__device__ int wphase_attempt(const StepParams &P, CellBuf<Real> &B, WarpShared &sh, double *usplit,
                              uint32_t gcell, trmcr_coll_rec *log, unsigned long long *log_count,
                              int64_t log_cap) {
  const int lane = threadIdx.x & 31;
  const RngKey K{P.k0, P.k1, gcell, P.step};
  const int n = sh.n;
  Perm pi0;
  pi0.rk = sh.pk; pi0.D = sh.D0;
  const int attempt = sh.r;
  PHASE_MARK(t_ph);
  wplan_counts<Real>(K, B, sh);
  WPHASE_ADD(1, t_ph);   // plan counts
  if (sh.flag != kOk) return sh.flag;
  wplan_execute<Real, WB, MOD>(P, K, B, sh, pi0, (Real)sh.sig_run, log, log_count, log_cap);
  WPHASE_ADD(2, t_ph);   // plan execute
  if (lane == 0) {
    if (attempt == 0) {
      sh.Ltot = sh.L;
      sh.U = B.Q[0] < n - sh.Ltot ? B.Q[0] : n - sh.Ltot;
      sh.nT = n - sh.Ltot - sh.U;
      sh.m_next = sh.m_cur;
      sh.S_est = sh.S0; sh.E1 = 0.0;
    } else {
      sh.Ltot += sh.L; sh.nT -= sh.L;
    }
    sh.done = 1;
  }
  __syncwarp();
  if (!P.adaptive) return kOk;
  wrad_estimate<Real>(P, B, sh, pi0);
  WPHASE_ADD(3, t_ph);   // RAD estimate
  if (lane == 0) {
    for (;;) {
      if (sh.E1 > P.delta2 && sh.m_cur < P.m_cap) {
        const int m_new = 2 * sh.m_cur < P.m_cap ? 2 * sh.m_cur : P.m_cap;
        wsplit_extend(K, sh, m_new, B.Q, B.L_cap, usplit);
        sh.r += 1;
        sh.lo = sh.m_cur + 1;
        sh.hi = sh.d < B.L_cap ? sh.d : B.L_cap;
        sh.budget = sh.nT;
        sh.leaf_off = sh.Ltot;
        sh.m_cur = m_new;
        sh.done = 0;
        if (sh.flag != kOk) break;
        // a retry whose plan is empty (no quota on the new levels) changes
        // nothing - same Theta, same estimate: it is counted and decided here
        int top = sh.hi;
        while (top >= sh.lo && B.Q[top] == 0) top--;
        if (top >= sh.lo && top >= 1) break;
        sh.done = 1;
      } else {
        sh.m_next = (sh.E1 < P.delta1) ? (sh.m_cur / 2 > 1 ? sh.m_cur / 2 : 1) : sh.m_cur;
        break;
      }
    }
  }
  __syncwarp();
  return sh.flag;
}

template <typename Real, bool WB>
__device__ void wphase_end(const StepParams &P, CellBuf<Real> &B, WarpShared &sh, Real *out_x, Real *out_y,
                           Real *out_z, uint32_t gcell, int32_t *m_state, double *stats_row) {
  const int lane = threadIdx.x & 31;
  const RngKey K{P.k0, P.k1, gcell, P.step};
  const int n = sh.n;
  Perm pi0;
  pi0.rk = sh.pk; pi0.D = sh.D0;
  // ---- A8 ----
  wmaxwellian<Real, WB>(P, K, B, sh, pi0, sh.c2);
  if (out_x != B.vx)
    for (int i = lane; i < n; i += 32) { out_x[i] = B.vx[i]; out_y[i] = B.vy[i]; out_z[i] = B.vz[i]; }
  if (lane == 0) {
    if (P.adaptive) *m_state = sh.m_next;
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
  __syncwarp();
}

// The cell (already staged in B.v*, n particles, sums of the staging pass in
// sx, sy, sz) through A3-A8, phases back to back.  Returns kOk or kOverflow
// (nothing written then except B's scratch).  Writes m_state, stats, and the
// velocities (out_* unless they alias the slab).
template <typename Real, bool WB, int MOD = -1>
__device__ int process_cell_warp(const StepParams &P, CellBuf<Real> &B, WarpShared &sh, double *usplit,
                                 double sx, double sy, double sz, Real *out_x, Real *out_y, Real *out_z, int n,
                                 uint32_t gcell, int32_t *m_state, double *stats_row, trmcr_coll_rec *log,
                                 unsigned long long *log_count, int64_t log_cap) {
  int rc = wphase_begin<Real, MOD>(P, B, sh, usplit, sx, sy, sz, n, gcell, m_state);
  if (rc != kOk) return rc;
  for (;;) {
    rc = wphase_attempt<Real, WB, MOD>(P, B, sh, usplit, gcell, log, log_count, log_cap);
    if (rc != kOk) return rc;
    if (sh.done) break;
  }
  wphase_end<Real, WB>(P, B, sh, out_x, out_y, out_z, gcell, m_state, stats_row);
  return kOk;
}

}  // namespace trmcr
