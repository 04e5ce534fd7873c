// shock.cuh — 1D stationary shock: reservoirs + free transport (A1) and the
// stable counting sort by cell (A2), fused with the per-cell collision step.
//
// Step (all on the context stream, no host round trip):
//   shock_prologue / ghost_gen   ghost slabs [x_min-Lg, x_min) and [x_max, x_max+Lg),
//                             Lg = (|u_B| + 6 sqrt(T_B)) dt, refilled with
//                             IR(rho_B Lg / w) particles of M(rho_B,u_B,T_B) [R26];
//                             transported; survivors counted per destination cell
//   transport_kernel          x <- x + v_x dt (splitting); destination
//                             cell; per-cell counts; displacement bound W
//   scan_offsets              exclusive scan -> new offsets (capacity check)
//   edge_place                ghosts + immigrants (few) placed at their stable
//                             positions at the ends of their cells
//   scatter_sorted            interior particles placed at their stable
//                             positions: tile histograms from transport_kernel,
//                             look-back over earlier tiles, in-tile ranks
//   shock_collide_warp        per cell, in place on the sorted arrays
//   shock_collide_smem/gmem   deferred cells: stable gather of their
//                             particles from the source window [c-W, c+W] in
//                             canonical order (left ghosts, interior in array
//                             order, right ghosts), then the collision step
//                             (cell_step.cuh) with rho_c = n_c w / dx, written
//                             to the other buffer.
#pragma once
#include "ctx.cuh"
#include "cell_warp.cuh"
#include "thermal.cuh"

namespace trmcr {

// Geometry seen by one rank: local cells [0, C) are global cells
// [cbase, cbase + C) of a Cg-cell grid on the GLOBAL domain [x_min, x_max).
struct ShockDev {
  int C, Cg, cbase;
  int has_left, has_right;     // a neighbouring slab exists (else: reservoir)
  double x_min, x_max, inv_dx, dt;
  float x_min_f, x_max_f;      // smallest floats >= x_min, x_max: for a float x, x >= x_min_f <=> (double)x >= x_min (same for x_max)
  double rho[2], u[2], T[2], Lg[2], y[2];
  int cap_g;
  int64_t cap;                 // particle capacity of the buffers: no store at or beyond it
  int64_t n_hint;              // a count the array is expected to exceed (15/16 of the last count the host saw): tiles
                               // below it load their particles before the step's true count has been read (a hint
                               // only: tiles above it read the count first, the result is the same)
};

constexpr int kDropped = INT32_MIN;   // destination of a particle that left the domain

// global cell of a position inside the domain, clamped (A2)
__device__ __forceinline__ int cell_of(const ShockDev &S, double x) {
  const double f = floor((x - S.x_min) * S.inv_dx);
  return f < 0.0 ? 0 : (f >= (double)S.Cg ? S.Cg - 1 : (int)f);
}

// Exchange buffer (caller memory, see trmcr_shock_set_exchange):
// [int32 count | pad to 16 B][cap x][cap vx][cap vy][cap vz][cap int32 global dest]
template <typename Real>
struct XBuf {
  int *count;
  Real *x, *vx, *vy, *vz;
  int32_t *dest;
  __host__ __device__ static XBuf bind(void *base, int cap) {
    XBuf b;
    unsigned char *p = reinterpret_cast<unsigned char *>(base);
    b.count = reinterpret_cast<int *>(p);
    Real *r = reinterpret_cast<Real *>(p + 16);
    b.x = r; b.vx = r + cap; b.vy = r + 2 * (size_t)cap; b.vz = r + 3 * (size_t)cap;
    b.dest = reinterpret_cast<int32_t *>(r + 4 * (size_t)cap);
    return b;
  }
  static size_t bytes(int cap) { return 16 + (size_t)cap * (4 * sizeof(Real) + 4); }
};

template <typename Real> __device__ __forceinline__ Real add_rn(Real a, Real b);
template <> __device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
template <> __device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
template <typename Real> __device__ __forceinline__ Real mul_rn(Real a, Real b);
template <> __device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
template <> __device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }

// A1 for one particle: x' = x + v_x dt (no FMA, [R29]) and its local
// destination cell (kDropped when it left the domain; may lie in a neighbour
// slab).  transport_kernel stores the destination cell but not x': the kernels
// that move the particles (scatter, gather, emigrant packing) read x and v_x
// anyway and recompute x' - the same arithmetic, so the same value - which
// saves the 4-byte write of x' per particle.  (Recomputing the destination
// there too, instead of storing it, measured slower: C5 scatter 0.50 ->
// 0.57 ms for 26 us less transport.)
template <typename Real>
__device__ __forceinline__ Real moved_x(const ShockDev &S, Real x, Real vx) {
  return add_rn<Real>(x, mul_rn<Real>(vx, (Real)S.dt));
}
template <typename Real>
__device__ __forceinline__ int dest_of(const ShockDev &S, Real xn) {
  const double xd = (double)xn;
  return (xd >= S.x_min && xd < S.x_max) ? cell_of(S, xd) - S.cbase : kDropped;
}
// The same value without branches (the transport's inner loop): the domain test
// on float thresholds for fp32 positions (exactly the double test, see
// ShockDev), floor by the conversion's rounding mode (the argument is >= 0 for a
// particle inside the domain), the upper clamp of cell_of as an integer min.
template <typename Real>
__device__ __forceinline__ int dest_of_fast(const ShockDev &S, Real xn) {
  const double xd = (double)xn;
  bool inside;
  if constexpr (sizeof(Real) == 4) inside = xn >= S.x_min_f && xn < S.x_max_f;
  else inside = xd >= S.x_min && xd < S.x_max;
  const int c = min(__double2int_rd((xd - S.x_min) * S.inv_dx), S.Cg - 1) - S.cbase;
  return inside ? c : kDropped;
}

// warp-aggregated atomicAdd(&counts[key], 1) for lanes with key >= 0
__device__ __forceinline__ void count_key(int32_t *counts, int key) {
  const unsigned act = 0xffffffffu;   // called by full warps
  const unsigned peers = __match_any_sync(act, key);
  const int lane = threadIdx.x & 31;
  if (key >= 0 && (__ffs(peers) - 1) == lane) atomicAdd(&counts[key], __popc(peers));
}

// ---- init: check the particles lie in the domain, sorted by cell; count ----
template <typename Real>
__global__ void shock_bin_init(ShockDev S, const Real *__restrict__ x, int64_t n, int32_t *counts, int *err) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int key = -1;                                  // full warps reach count_key (warp-aggregated:
  if (i < n) {                                   // sorted input, a warp's particles share few cells)
    const double xi = (double)x[i];
    if (!(xi >= S.x_min && xi < S.x_max)) {
      atomicOr(err, 4);
    } else {
      const int c = cell_of(S, xi) - S.cbase;
      if (c < 0 || c >= S.C) atomicOr(err, 4);
      else key = c;
      if (i > 0 && cell_of(S, (double)x[i - 1]) - S.cbase > c) atomicOr(err, 8);
    }
  }
  count_key(counts, key);
}

// exclusive scan of counts[0..C) into off[0..C], off[C] = total (one CTA).
// Each thread owns 16 consecutive counts: 4 int4 loads and 8 longlong2 stores
// (16-byte I/O) on full rounds, scalar on the ragged last one.
__global__ void __launch_bounds__(1024) scan_offsets(const int32_t *__restrict__ counts, int C, int64_t *off,
                                                     int64_t cap, int *err) {
  pdl_wait();   // no-op without programmatic dependent launch
  __shared__ int64_t wsum[32];
  __shared__ int64_t carry;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int ITEMS = 16;
  if (tid == 0) carry = 0;
  __syncthreads();
  const bool al = ((reinterpret_cast<uintptr_t>(counts) | reinterpret_cast<uintptr_t>(off)) & 15) == 0;
  for (int base = 0; base < C; base += 1024 * ITEMS) {
    const int i0 = base + tid * ITEMS;
    const bool vec = al && i0 + ITEMS <= C;
    int v[ITEMS];
    if (vec) {
#pragma unroll
      for (int q = 0; q < ITEMS / 4; ++q) {
        const int4 w = *reinterpret_cast<const int4 *>(counts + i0 + 4 * q);
        v[4 * q] = w.x; v[4 * q + 1] = w.y; v[4 * q + 2] = w.z; v[4 * q + 3] = w.w;
      }
    } else {
#pragma unroll
      for (int k = 0; k < ITEMS; ++k) v[k] = i0 + k < C ? counts[i0 + k] : 0;
    }
    int64_t s = 0;
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) s += v[k];
    int64_t incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      int64_t w = wsum[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t t = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += t;
      }
      wsum[lane] = w;
    }
    __syncthreads();
    int64_t run = carry + (warp > 0 ? wsum[warp - 1] : 0) + incl - s;
    if (vec) {
#pragma unroll
      for (int q = 0; q < ITEMS / 2; ++q) {
        const int64_t a = run;
        run += v[2 * q];
        const int64_t b = run;
        run += v[2 * q + 1];
        *reinterpret_cast<longlong2 *>(off + i0 + 2 * q) = make_longlong2(a, b);
      }
    } else {
#pragma unroll
      for (int k = 0; k < ITEMS; ++k) {
        if (i0 + k < C) off[i0 + k] = run;
        run += v[k];
      }
    }
    __syncthreads();
    if (tid == 0) carry += wsum[31];
    __syncthreads();
  }
  if (tid == 0) {
    off[C] = carry;
    if (carry > cap) atomicOr(err, 2);
  }
  pdl_trigger();
}

// Multi-CTA exclusive scan with decoupled look-back: CTA b scans its 4096
// counts, publishes its aggregate, then adds the predecessors' aggregates
// (or the first inclusive prefix it meets) and publishes its own inclusive
// prefix.  Status words: epoch (bits 34+) | flag (bits 32-33: 1 aggregate,
// 2 inclusive prefix) | value (bits 0-31; totals stay below 2^31) - stamped
// with a per-call epoch, so nothing needs zeroing between calls.  Every CTA
// is resident at once (a few dozen at most), so the spin-waits progress.
constexpr int kScanThreads = 256, kScanItems = 16, kScanTile = kScanThreads * kScanItems;
// 30-bit stamps, never 0 (the status words start zeroed)
inline uint32_t next_scan_epoch(ShockState &s) {
  s.scan_epoch = (s.scan_epoch + 1u) & 0x3FFFFFFFu;
  if (s.scan_epoch == 0u) s.scan_epoch = 1u;
  return s.scan_epoch;
}
__global__ void __launch_bounds__(kScanThreads) scan_offsets_lb(const int32_t *__restrict__ counts, int C,
                                                                int64_t *off, int64_t cap, int *err,
                                                                unsigned long long *status, uint32_t epoch) {
  pdl_wait();   // programmatic dependent launch: the predecessor's writes are visible
  __shared__ int64_t wsum[kScanThreads / 32];
  __shared__ int64_t s_excl;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, b = blockIdx.x;
  const int i0 = b * kScanTile + tid * kScanItems;
  const bool vec = ((reinterpret_cast<uintptr_t>(counts) | reinterpret_cast<uintptr_t>(off)) & 15) == 0 &&
                   i0 + kScanItems <= C;
  int v[kScanItems];
  if (vec) {
#pragma unroll
    for (int q = 0; q < kScanItems / 4; ++q) {
      const int4 w = *reinterpret_cast<const int4 *>(counts + i0 + 4 * q);
      v[4 * q] = w.x; v[4 * q + 1] = w.y; v[4 * q + 2] = w.z; v[4 * q + 3] = w.w;
    }
  } else {
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) v[k] = i0 + k < C ? counts[i0 + k] : 0;
  }
  int64_t sum = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) sum += v[k];
  int64_t incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int64_t w = lane < kScanThreads / 32 ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t t = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += t;
    }
    if (lane < kScanThreads / 32) wsum[lane] = w;
    const int64_t agg = __shfl_sync(0xffffffffu, w, kScanThreads / 32 - 1);
    const unsigned long long tag = (unsigned long long)epoch << 34;
    int64_t excl = 0;
    if (b == 0) {
      if (lane == 0) atomicExch(&status[0], tag | (2ull << 32) | (unsigned long long)agg);
    } else {
      if (lane == 0) atomicExch(&status[b], tag | (1ull << 32) | (unsigned long long)agg);
      // look back over the predecessors, 32 at a time
      for (int j0 = b - 1;; j0 -= 32) {
        const int j = j0 - lane;
        unsigned long long st = 0;
        if (j >= 0) {
          do {
            st = atomicAdd(&status[j], 0ull);
          } while ((st >> 34) != (unsigned long long)epoch || ((st >> 32) & 3ull) == 0ull);
        }
        const bool pre = j >= 0 && ((st >> 32) & 3ull) == 2ull;
        const unsigned pm = __ballot_sync(0xffffffffu, pre);
        const int stop = pm ? __ffs(pm) - 1 : 32;     // first inclusive prefix (nearest predecessor)
        int64_t add = (j >= 0 && lane <= stop) ? (int64_t)(st & 0xFFFFFFFFull) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) add += __shfl_xor_sync(0xffffffffu, add, o);
        excl += add;
        if (pm || j0 - 31 <= 0) break;
      }
      if (lane == 0)
        atomicExch(&status[b], tag | (2ull << 32) | (unsigned long long)(excl + agg));
    }
    if (lane == 0) {
      s_excl = excl;
      if (b == (int)gridDim.x - 1) {
        off[C] = excl + agg;
        if (excl + agg > cap) atomicOr(err, 2);
      }
    }
  }
  __syncthreads();
  int64_t run = s_excl + (warp > 0 ? wsum[warp - 1] : 0) + incl - sum;
  if (vec) {
#pragma unroll
    for (int q = 0; q < kScanItems / 2; ++q) {
      const int64_t a = run;
      run += v[2 * q];
      const int64_t c2 = run;
      run += v[2 * q + 1];
      *reinterpret_cast<longlong2 *>(off + i0 + 2 * q) = make_longlong2(a, c2);
    }
  } else {
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
      if (i0 + k < C) off[i0 + k] = run;
      run += v[k];
    }
  }
  pdl_trigger();
}

// ---- A1: reservoir ghost counts IR(rho_B Lg / w) ----
// First kernel of a shock step: zeroes the step's destination counts, window
// bounds, accounting and overflow counter (one launch instead of four memsets)
// and draws the number of reservoir ghosts per side.
__global__ void __launch_bounds__(256) shock_prologue(ShockDev S, uint32_t k0, uint32_t k1, uint32_t step, int *ng,
                                                      int *err, int32_t *counts, int *W, unsigned long long *acct,
                                                      int *ovf_count, int *defer_count, int *far_cnt_next) {
  pdl_wait();   // programmatic dependent launch: the predecessor's writes are visible
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < S.C; i += gridDim.x * blockDim.x) counts[i] = 0;
  if (blockIdx.x != 0) return;
  if (threadIdx.x < 3) W[threadIdx.x] = 0;
  if (threadIdx.x < 4) acct[threadIdx.x] = 0ull;
  if (threadIdx.x == 4) *ovf_count = 0;
  if (threadIdx.x == 5) *defer_count = 0;
  if (threadIdx.x == 6 && far_cnt_next) *far_cnt_next = 0;   // fused step: the far list this step writes
  const int side = threadIdx.x;
  if (side > 1) return;
  if (side == 0 ? S.has_left : S.has_right) { ng[side] = 0; return; }   // a neighbour, not a reservoir
  const RngKey K{k0, k1, 0xFFFFFFF0u + (uint32_t)side, step};
  const uint4 w = K(kResv, side, 0, 0);
  const double y = S.y[side];
  const double fl = floor(y);
  int64_t N = (int64_t)fl + ((u53(w.x, w.y) < y - fl) ? 1 : 0);
  if (N > S.cap_g) { atomicOr(err, 2); N = S.cap_g; }
  ng[side] = (int)N;
  pdl_trigger();
}

// ---- A1: ghost particles, transported; survivors counted ----
template <typename Real>
__global__ void ghost_gen(ShockDev S, uint32_t k0, uint32_t k1, uint32_t step, const int *ng, Real *gx0,
                          Real *gx1, Real *gvx0, Real *gvy0, Real *gvz0, Real *gvx1, Real *gvy1, Real *gvz1,
                          int32_t *gd0, int32_t *gd1, int32_t *counts, int *W, unsigned long long *acct) {
  pdl_wait();   // programmatic dependent launch: the predecessor's writes are visible
  const int side = blockIdx.y;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= ng[side]) return;
  const RngKey K{k0, k1, 0xFFFFFFF0u + (uint32_t)side, step};
  const uint4 a = K(kResv, side, 1, k), b = K(kResv, side, 2, k), c = K(kResv, side, 3, k);
  const double upos = u53(a.x, a.y), u1 = u53(a.z, a.w), u2 = u53(b.x, b.y), u3 = u53(b.z, b.w);
  const double u4 = u53(c.x, c.y);
  const double Lg = S.Lg[side];
  const double xg = side ? __dadd_rn(S.x_max, __dmul_rn(Lg, upos))
                         : __dadd_rn(__dsub_rn(S.x_min, Lg), __dmul_rn(Lg, upos));
  const double r1 = sqrt(-2.0 * log(u1)), r3 = sqrt(-2.0 * log(u3));
  double s2, c2, s4, c4;
  sincospi(2.0 * u2, &s2, &c2);
  sincospi(2.0 * u4, &s4, &c4);
  const double sT = sqrt(S.T[side]);
  const Real vx = (Real)(S.u[side] + sT * (r1 * c2));
  const Real vy = (Real)(sT * (r1 * s2));
  const Real vz = (Real)(sT * (r3 * c4));
  const Real xn = add_rn<Real>((Real)xg, mul_rn<Real>(vx, (Real)S.dt));
  const double xd = (double)xn;
  const bool keep = xd >= S.x_min && xd < S.x_max;
  const int d = keep ? cell_of(S, xd) - S.cbase : kDropped;   // local (may lie in a neighbour)
  Real *gx = side ? gx1 : gx0;
  Real *gvx = side ? gvx1 : gvx0, *gvy = side ? gvy1 : gvy0, *gvz = side ? gvz1 : gvz0;
  int32_t *gd = side ? gd1 : gd0;
  gx[k] = xn; gvx[k] = vx; gvy[k] = vy; gvz[k] = vz; gd[k] = d;
  if (keep) {
    atomicAdd(&acct[side], 1ull);
    if (d >= 0 && d < S.C) {
      atomicAdd(&counts[d], 1);
      atomicMax(W, side ? S.C - d : d + 1);
    } else {
      atomicMax(W + 1, S.C + 1);   // emigrating ghost: pack kernel scans the ghosts
    }
  }
  pdl_trigger();
}

// ---- A1: free transport of the interior particles ----
// dest = local destination cell (outside [0, C): emigrant to a neighbouring
// slab; kDropped: left the domain).  The particles of one CTA are sorted by
// source cell and move less than a cell or two, so their destinations fall in
// a small window: counts are accumulated in a shared-memory histogram over
// [dmin, dmin + kHist) and flushed with one global atomic per touched cell
// (a destination outside the window falls back to a global atomic).
// W[0] = bound of the local displacements, W[1] = emigrant scan width, acct[2] = dropped.
// Large problems: tiles of 256 x 4 x TRMCR_TILE_GROUPS particles.  Measured on C5 with the
// scatter's CTA size (transport + scatter, ms): 4 groups / 512 threads 0.152 + 0.465, 4 / 256
// 0.152 + 0.511, 4 / 1024 0.152 + 0.769, 3 / 512 0.154 + 0.431, 3 / 256 0.154 + 0.487, 5 / 512
// 0.154 + 0.443, 2 / 512 0.162 + 0.510, 2 / 256 0.162 + 0.420 (chosen), 1 / 256 0.203 + 0.447.
#ifndef TRMCR_TILE_GROUPS
#define TRMCR_TILE_GROUPS 2
#endif
constexpr int kTransportThreads = 256, kTransportPer = 4, kTransportGroups = TRMCR_TILE_GROUPS, kHist = 256;
// particles per transport tile: thread t of the CTA owns the 4-particle groups
// t, t + 256, t + 512, t + 768 of the tile (16-byte coalesced I/O)
constexpr int kTile = kTransportThreads * kTransportPer * kTransportGroups;   // large problems
__host__ __device__ constexpr int tile_of(int ng) { return kTransportThreads * kTransportPer * ng; }
constexpr int kEdgeBins = 4096;   // cells from a domain / slab edge that ghosts and immigrants may reach
constexpr int kEmigrantCells = 64;   // cells from a neighbour within which an emigrant may start (else error 256)

template <typename Real, int NG>
__global__ void __launch_bounds__(kTransportThreads)
transport_kernel(ShockDev S, const int64_t *__restrict__ off_old, Real *x, const Real *__restrict__ vx,
                 int32_t *dest, int32_t *counts, int *W, unsigned long long *acct, int32_t *tileH, int2 *tile_meta,
                 int phase, int *err) {
  pdl_wait();   // programmatic dependent launch: the predecessor's writes are visible
  constexpr int P4 = kTransportPer, TILE = tile_of(NG);
  // Slabs with neighbours transport in two launches: phase 1 takes the tiles
  // that hold particles of the kEmigrantCells cells next to a neighbour (the
  // only possible sources of emigrants), so the emigrants can be packed and
  // their exchange started while phase 2 transports the bulk.  phase 0: every
  // tile (no neighbour).  A tile is of one kind in both launches (same test).
  if (phase != 0) {
    const int El = S.has_left ? min(kEmigrantCells, S.C) : 0, Er = S.has_right ? min(kEmigrantCells, S.C) : 0;
    const int64_t t0 = (int64_t)blockIdx.x * TILE;
    const bool edge = (El > 0 && t0 < off_old[El]) || (Er > 0 && t0 + TILE > off_old[S.C - Er]);
    if (edge != (phase == 1)) { pdl_trigger(); return; }
  }
  __shared__ int s_hist[kHist];
  __shared__ int s_red[4][kTransportThreads / 32];
  __shared__ int s_dmin;
  const int64_t n = off_old[S.C];
  const int64_t tile0 = (int64_t)blockIdx.x * TILE;
  const bool spec = tile0 + TILE <= S.n_hint && tile0 + TILE <= S.cap;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ Real s_xend[2];
  int d[NG][P4];
  int dropped = 0, dmin = INT32_MAX, dmax = -1, lemi = 0, remi = 0;
  // every load of the tile first, then the arithmetic (x and v are read only:
  // the moves are recomputed where the particles are moved)
  Real xa[NG][P4], va[NG][P4];
#pragma unroll
  for (int g = 0; g < NG; ++g) {
    const int64_t i0 = tile0 + ((int64_t)g * kTransportThreads + threadIdx.x) * P4;
    // tiles below the hint: bounded by the buffers' capacity, not by n, so the loads do not
    // wait for n's (slots beyond n would be read and never used)
    const int64_t lim = spec ? S.cap : n;
    if ((i0 + P4 <= lim) && (sizeof(Real) * P4 == 16)) {
      using V = typename Vec<Real>::T;
      const V xv = *reinterpret_cast<const V *>(x + i0), vv = *reinterpret_cast<const V *>(vx + i0);
#pragma unroll
      for (int k = 0; k < P4; ++k) { xa[g][k] = vget<V, Real>(xv, k); va[g][k] = vget<V, Real>(vv, k); }
    } else {
#pragma unroll
      for (int k = 0; k < P4; ++k) {
        xa[g][k] = (i0 + k < lim) ? x[i0 + k] : Real(0);
        va[g][k] = (i0 + k < lim) ? vx[i0 + k] : Real(0);
      }
    }
  }
  // source cells of the tile's first and last particles (the array is sorted
  // by cell: every source cell of the tile lies between them)
  if (threadIdx.x == 0 && tile0 < n) {
    s_xend[0] = x[tile0];
    s_xend[1] = x[min(n, tile0 + (int64_t)TILE) - 1];
  }
  __syncthreads();
  // every slot of a full tile holds a particle (uniform test): its copy of the loop has no bound checks
  auto classify = [&](auto FULL) {
    constexpr bool full = decltype(FULL)::value;
#pragma unroll
    for (int g = 0; g < NG; ++g) {
      const int64_t i0 = tile0 + ((int64_t)g * kTransportThreads + threadIdx.x) * P4;
      const bool vec = full || ((i0 + P4 <= n) && (sizeof(Real) * P4 == 16));
      int dl[P4];
#pragma unroll
      for (int k = 0; k < P4; ++k) {          // no branches: a slot beyond n counts as nothing
        const bool on = full || i0 + k < n;
        dl[k] = dest_of_fast<Real>(S, moved_x<Real>(S, xa[g][k], va[g][k]));
        const bool local = on && (unsigned)dl[k] < (unsigned)S.C;
        dropped += (on && dl[k] == kDropped) ? 1 : 0;
        dmin = min(dmin, local ? dl[k] : INT32_MAX);
        dmax = max(dmax, local ? dl[k] : -1);
        lemi |= (on && dl[k] < 0 && dl[k] != kDropped) ? 1 : 0;
        remi |= (on && dl[k] >= S.C) ? 1 : 0;
        d[g][k] = local ? dl[k] : -1;         // counted below: local only
      }
      if (vec) *reinterpret_cast<int4 *>(dest + i0) = make_int4(dl[0], dl[1], dl[2], dl[3]);
      else {
#pragma unroll
        for (int k = 0; k < P4; ++k) if (i0 + k < n) dest[i0 + k] = dl[k];
      }
    }
  };
  if (tile0 + TILE <= n && sizeof(Real) * P4 == 16) classify(std::true_type{});
  else classify(std::false_type{});
  // CTA reductions: destination window, emigrant sides, dropped.  With the
  // tile's source cells in [s0, s1], W[0] = max(dmax - s0, s1 - dmin) bounds
  // every local displacement and W[1] = s1 + 1 (left) / C - s0 (right) every
  // emigrant's source distance from the edge (bounds: wider scans, same result)
  dmin = __reduce_min_sync(0xffffffffu, dmin);
  const int wdx = __reduce_max_sync(0xffffffffu, dmax);
  const int wl = __reduce_or_sync(0xffffffffu, lemi), wr = __reduce_or_sync(0xffffffffu, remi);
  const int wdr = __reduce_add_sync(0xffffffffu, dropped);
  if (threadIdx.x < kHist) s_hist[threadIdx.x] = 0;
  if (lane == 0) { s_red[0][warp] = dmin; s_red[1][warp] = wdx; s_red[2][warp] = wl; s_red[3][warp] = wr; }
  __syncthreads();
  if (threadIdx.x == 0) {
    int m = INT32_MAX, mx = -1, l = 0, r = 0;
    for (int w = 0; w < kTransportThreads / 32; ++w) {
      m = min(m, s_red[0][w]); mx = max(mx, s_red[1][w]); l |= s_red[2][w]; r |= s_red[3][w];
    }
    s_dmin = m;
    const int s0 = tile0 < n ? cell_of(S, (double)s_xend[0]) - S.cbase : 0;
    const int s1 = tile0 < n ? cell_of(S, (double)s_xend[1]) - S.cbase : -1;
    if (tile_meta) tile_meta[blockIdx.x] = make_int2(m, s1);
    const int md = mx >= 0 ? max(mx - s0, s1 - m) : 0;
    const int me = max(l ? s1 + 1 : 0, r ? S.C - s0 : 0);
    if (md > 0 && md > *((volatile int *)W)) atomicMax(W, md);
    if (me > 0 && me > *((volatile int *)(W + 1))) atomicMax(W + 1, me);
    if (phase == 2 && (l || r)) atomicOr(err, 256);   // an emigrant from the bulk: already packed without it
  }
  if (lane == 0 && wdr) atomicAdd(&acct[2], (unsigned long long)wdr);
  __syncthreads();
  const int base = s_dmin;
#pragma unroll
  for (int g = 0; g < NG; ++g)
#pragma unroll
    for (int k = 0; k < P4; ++k) {
      if (d[g][k] < 0) continue;
      const int h = d[g][k] - base;
      if (h < kHist) atomicAdd(&s_hist[h], 1);
      else { atomicAdd(&counts[d[g][k]], 1); if (tileH) W[2] = 1; }   // scatter sort not possible this step
    }
  __syncthreads();
  if (threadIdx.x < kHist) {
    const int h = s_hist[threadIdx.x];
    if (h > 0) atomicAdd(&counts[base + threadIdx.x], h);
    if (tileH) tileH[(size_t)blockIdx.x * kHist + threadIdx.x] = h;
  }
  pdl_trigger();
}

// ---- slab exchange: pack emigrants (stable, canonical order) ----
// side 0: destination left of the slab (dest < 0), side 1: right (dest >= C).
// Canonical source order: left ghosts, interior (array order), right ghosts.
// One CTA per side; blockDim*8 entries per round, CTA scan for positions.
template <typename Real>
__global__ void __launch_bounds__(1024)
pack_emigrants(ShockDev S, const int64_t *__restrict__ off_old, const int *ng, const int *W, const Real *x,
               const Real *vx, const Real *vy, const Real *vz, const int32_t *dest, const Real *gx0,
               const Real *gvx0, const Real *gvy0, const Real *gvz0, const int32_t *gd0, const Real *gx1,
               const Real *gvx1, const Real *gvy1, const Real *gvz1, const int32_t *gd1, void *send_l,
               void *send_r, int cap, int *err, int tile) {
  pdl_wait();   // programmatic dependent launch: the predecessor's writes are visible
  constexpr int R = 8;
  __shared__ int wcnt[32];
  const int side = blockIdx.x;
  if (side == 0 ? !S.has_left : !S.has_right) return;
  XBuf<Real> B = XBuf<Real>::bind(side == 0 ? send_l : send_r, cap);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int We = W[1];
  int running = 0;
  for (int seg = 0; seg < 3; ++seg) {
    int64_t lo, hi;
    const Real *sx, *svx, *svy, *svz;
    const int32_t *sd;
    if (seg == 1) {
      if (We <= 0) continue;
      const int a = side == 0 ? 0 : max(S.C - We, 0), b = side == 0 ? min(We, S.C) : S.C;
      lo = off_old[a]; hi = off_old[b];
      // only the edge tiles have been transported (transport_kernel phase 1): stay inside them
      // (an emigrant beyond them is reported by phase 2, error 256)
      if (side == 0) hi = min(hi, (off_old[min(kEmigrantCells, S.C)] + tile - 1) / tile * tile);
      else lo = max(lo, off_old[S.C - min(kEmigrantCells, S.C)] / tile * tile);
      sx = x; svx = vx; svy = vy; svz = vz; sd = dest;
    } else {
      const int g = seg == 0 ? 0 : 1;
      lo = 0; hi = ng[g];
      sx = g ? gx1 : gx0; svx = g ? gvx1 : gvx0; svy = g ? gvy1 : gvy0; svz = g ? gvz1 : gvz0;
      sd = g ? gd1 : gd0;
    }
    for (int64_t b0 = lo; b0 < hi; b0 += (int64_t)blockDim.x * R) {
      const int64_t i0 = b0 + (int64_t)tid * R;
      unsigned bits = 0;
#pragma unroll
      for (int k = 0; k < R; ++k) {
        const int64_t i = i0 + k;
        if (i < hi) {
          const int dd = sd[i];
          const bool m = dd != kDropped && (side == 0 ? dd < 0 : dd >= S.C);
          if (m) bits |= 1u << k;
        }
      }
      const int mine = __popc(bits);
      int incl = mine;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      if (lane == 31) wcnt[warp] = incl;
      __syncthreads();
      int wb = 0, tot = 0;
      for (int w = 0; w < nw; ++w) { const int t = wcnt[w]; wb += (w < warp) ? t : 0; tot += t; }
      int pos = running + wb + incl - mine;
      while (bits) {
        const int k = __ffs(bits) - 1;
        bits &= bits - 1;
        const int64_t i = i0 + k;
        if (pos < cap) {
          const Real xn = seg == 1 ? moved_x<Real>(S, sx[i], svx[i]) : sx[i];
          B.x[pos] = xn; B.vx[pos] = svx[i]; B.vy[pos] = svy[i]; B.vz[pos] = svz[i];
          B.dest[pos] = sd[i] + S.cbase;   // global destination cell
        }
        ++pos;
      }
      running += tot;
      __syncthreads();
    }
  }
  if (tid == 0) {
    if (running > cap) { atomicOr(err, 2); running = cap; }
    *B.count = running;
  }
  pdl_trigger();
}

// ---- slab exchange: immigrants (received) join the local counts ----
// side 0: from the left neighbour (virtual source before cell 0),
// side 1: from the right neighbour (virtual source after cell C-1).
template <typename Real>
__global__ void immigrant_count(ShockDev S, const void *recv_l, const void *recv_r, int cap, int32_t *counts,
                                int *W, int *err) {
  pdl_wait();   // programmatic dependent launch: the predecessor's writes are visible
  const int side = blockIdx.y;
  if (side == 0 ? !S.has_left : !S.has_right) return;
  const XBuf<Real> B = XBuf<Real>::bind(const_cast<void *>(side == 0 ? recv_l : recv_r), cap);
  const int n = min(*B.count, cap);
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int d = B.dest[k] - S.cbase;
  if (d < 0 || d >= S.C) { atomicOr(err, 32); return; }   // would need more than one hop
  atomicAdd(&counts[d], 1);
  atomicMax(W, side == 0 ? d + 1 : S.C - d);
  pdl_trigger();
}

// ---- A2 by scatter: ghosts and immigrants (canonical order) ----
// side 0: left reservoir ghosts, then left immigrants: the first particles of
// their cells, pos = off_new[d] + running count; lcnt[d] = how many (read by
// scatter_sorted).  side 1: right immigrants, then right reservoir ghosts: the
// last particles of their cells, pos = off_new[d + 1] - total[d] + running.
// One CTA per side: each round covers kEdgeThreads consecutive particles of a
// segment; the payload and off_new loads of all warps are in flight at once
// and only the running-count update is ordered (warp by warp, a short chain in
// shared memory), so the ranks are the index-order ones.
constexpr int kEdgeThreads = 512;
template <typename Real>
__global__ void __launch_bounds__(kEdgeThreads)
edge_place(ShockDev S, const int64_t *__restrict__ off_new, const int *ng, const void *recv_l, const void *recv_r,
           int xcap, const Real *gx0, const Real *gvx0, const Real *gvy0, const Real *gvz0, const int32_t *gd0,
           const Real *gx1, const Real *gvx1, const Real *gvy1, const Real *gvz1, const int32_t *gd1,
           int32_t *lcnt, Real *ox, Real *ovx, Real *ovy, Real *ovz, int *W) {
  pdl_wait();   // programmatic dependent launch: the predecessor's writes are visible
  constexpr int NW = kEdgeThreads / 32;
  __shared__ int run[kEdgeBins];
  __shared__ int turn;
  volatile int *vrun = run, *vturn = &turn;
  const int side = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int b = tid; b < kEdgeBins; b += kEdgeThreads) run[b] = 0;
  if (tid == 0) turn = 0;
  __syncthreads();
  // side 0 fills cells from their start, in index order: ghosts(0), then
  // immigrants(0).  Side 1 fills them from their end, backwards: the canonical
  // order there is immigrants(1), ghosts(1), so ghosts(1) come first, each
  // segment in reverse index order (no count pass needed).
  const bool back = side == 1;
  const int my_turn = back ? NW - 1 - warp : warp;                    // order of the warps in a round
  const unsigned rank_mask = back ? ~((2u << lane) - 1u) : ((1u << lane) - 1u);   // peers placed before
  for (int seg = 0; seg < 2; ++seg) {
    const bool ghosts = seg == 0;
    int cnt = 0, shift = 0;
    const Real *px, *pvx, *pvy, *pvz;
    const int32_t *pd;
    if (ghosts) {
      if (side == 0 ? S.has_left : S.has_right) continue;
      cnt = ng[side];
      px = side ? gx1 : gx0; pvx = side ? gvx1 : gvx0; pvy = side ? gvy1 : gvy0; pvz = side ? gvz1 : gvz0;
      pd = side ? gd1 : gd0;
    } else {
      const void *rb = side == 0 ? recv_l : recv_r;
      if (rb == nullptr) continue;
      const XBuf<Real> X = XBuf<Real>::bind(const_cast<void *>(rb), xcap);
      cnt = min(*X.count, xcap);
      px = X.x; pvx = X.vx; pvy = X.vy; pvz = X.vz; pd = X.dest;
      shift = S.cbase;                      // immigrants carry global destinations
    }
    for (int r0 = 0; r0 < cnt; r0 += kEdgeThreads) {
      const int k = back ? cnt - r0 - kEdgeThreads + tid : r0 + tid;
      int d = -1;
      if (k >= 0 && k < cnt) {
        const int dd = pd[k];
        if (dd != kDropped && dd - shift >= 0 && dd - shift < S.C) d = dd - shift;
      }
      const int bin = d < 0 ? -1 : (side == 0 ? d : S.C - 1 - d);
      if (bin >= kEdgeBins) W[2] = 1;     // out of reach of the edge bins: gather this step
      const bool ok = bin >= 0 && bin < kEdgeBins;
      const unsigned peers = __match_any_sync(0xffffffffu, ok ? bin : -1 - lane);
      const bool leader = __ffs(peers) - 1 == lane;
      Real a = Real(0), bx = Real(0), by = Real(0), bz = Real(0);
      int64_t base = 0;
      if (ok) {
        a = px[k]; bx = pvx[k]; by = pvy[k]; bz = pvz[k];
        base = back ? off_new[d + 1] - 1 : off_new[d];
      }
      // this warp's turn: every warp placed before it in this round has counted
      if (__any_sync(0xffffffffu, ok)) {
        if (lane == 0)
          while (*vturn != my_turn) {}
        __syncwarp();
        int r = 0, rank = 0;
        if (ok) { r = vrun[bin]; rank = r + __popc(peers & rank_mask); }
        __syncwarp();
        if (ok && leader) vrun[bin] = r + __popc(peers);
        __threadfence_block();
        __syncwarp();
        if (ok) {
          const int64_t pos = back ? base - rank : base + rank;
          if (pos >= 0 && pos < S.cap) { ox[pos] = a; ovx[pos] = bx; ovy[pos] = by; ovz[pos] = bz; }
        }
      } else if (lane == 0) {
        while (*vturn != my_turn) {}
      }
      if (lane == 0) *vturn = my_turn + 1;
      __syncthreads();
      if (tid == 0) turn = 0;
      __syncthreads();
    }
  }
  if (side == 0)
    for (int b = tid; b < kEdgeBins; b += kEdgeThreads) lcnt[b] = run[b];
  pdl_trigger();
}

// ---- A2 by scatter: interior particles ----
// Tile t = transport tile t (tile_of(NG) consecutive particles of the cell-sorted
// source array).  A particle's stable position in its destination cell d is
// off_new[d] + lcnt[d] + (particles of earlier tiles with destination d) +
// (its rank among the tile's particles with destination d, in index order).
// Earlier tiles are looked back over until one whose last source cell is more
// than W cells before the tile's first destination (none of its particles, nor
// any earlier one, can reach it); transport_kernel stored each tile's
// destination histogram over [dmin, dmin + kHist).
#ifndef TRMCR_SCATTER_THREADS
#define TRMCR_SCATTER_THREADS 256   // with the tile size, see TRMCR_TILE_GROUPS (round 1, tiles of 4096: 256 -> 0.62 ms, 1024 -> 0.69, 512 -> 0.50)
#endif
constexpr int kScatterThreads = TRMCR_SCATTER_THREADS;
template <typename Real, int NG>
__global__ void __launch_bounds__(kScatterThreads)
scatter_sorted(ShockDev S, const int64_t *__restrict__ off_old, const int64_t *__restrict__ off_new,
               const Real *__restrict__ x, const Real *__restrict__ vx, const Real *__restrict__ vy,
               const Real *__restrict__ vz, const int32_t *__restrict__ dest, const int32_t *__restrict__ tileH,
               const int2 *__restrict__ tile_meta, const int32_t *__restrict__ lcnt, const int *W,
               Real *__restrict__ ox, Real *__restrict__ ovx, Real *__restrict__ ovy, Real *__restrict__ ovz) {
  pdl_wait();   // programmatic dependent launch: the predecessor's writes are visible
  constexpr int NW = kScatterThreads / 32, PARTS = kScatterThreads / kHist;
  constexpr int TILE = tile_of(NG);
  constexpr int CHUNK = TILE / NW, ROUNDS = CHUNK / 32;   // each warp: CHUNK consecutive particles
  static_assert(ROUNDS >= 1, "tile smaller than the CTA");
  __shared__ int s_part[PARTS][kHist];
  __shared__ int s_wc[NW][kHist];                          // per-warp counts, then running positions
  __shared__ int64_t s_off[kHist];                         // off_new of the tile's destination cells
  __shared__ int2 s_meta[32];
  __shared__ int s_nb, s_more;
  // fp32: the tile's x, v_x, v_y, v_z are staged in shared memory by 1-D bulk
  // copies issued first, so the whole tile's reads are in flight while the
  // destinations are ranked (the data movement was bound by load latency:
  // 8 long-scoreboard stalls per issue with loads issued 4 rounds at a time)
  constexpr bool kStage = sizeof(Real) == 4;
  extern __shared__ __align__(16) unsigned char s_stage[];   // [4][TILE] Real when kStage
  __shared__ uint64_t s_bar;
  const int t = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t i_begin = (int64_t)t * TILE;
  Real *st_x = reinterpret_cast<Real *>(s_stage), *st_vx = st_x + TILE, *st_vy = st_vx + TILE, *st_vz = st_vy + TILE;
  // The bulk copies are sized by the buffers' capacity, not by the particle
  // count: below the hint they start before any load of this kernel has
  // returned (slots beyond the count are copied and never used).
  if (i_begin + TILE > S.n_hint && i_begin >= off_old[S.C]) return;   // (tiles beyond the hint read the count first)
  const int ccnt = (int)max((int64_t)0, min((int64_t)TILE, S.cap - i_begin));
  const int tbulk = (ccnt * (int)sizeof(Real)) & ~15;   // bytes per array through the bulk copy
  if constexpr (kStage) {
    if (tid == 0) {
      mbar_init(&s_bar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      mbar_expect_tx(&s_bar, 4u * (uint32_t)tbulk);
      if (tbulk > 0) {
        bulk_g2s(st_x, x + i_begin, (uint32_t)tbulk, &s_bar);
        bulk_g2s(st_vx, vx + i_begin, (uint32_t)tbulk, &s_bar);
        bulk_g2s(st_vy, vy + i_begin, (uint32_t)tbulk, &s_bar);
        bulk_g2s(st_vz, vz + i_begin, (uint32_t)tbulk, &s_bar);
      }
    }
  }
  // One round of loads: the step's scalars, this tile's and the 32 previous
  // tiles' metadata and this warp's destinations (tested afterwards - issued
  // one after the other, each paid its own latency: 4 of the tile's ~14).
  const int w2 = W[2], Wd = W[0];
  const int64_t tot = off_new[S.C], n = off_old[S.C];
  const int2 tmeta = tile_meta[t];
  int2 mprev = make_int2(INT32_MAX, -1);
  if (warp == 0 && t - 1 - lane >= 0) mprev = tile_meta[t - 1 - lane];
  const int64_t c0 = i_begin + (int64_t)warp * CHUNK;
  int bins[ROUNDS];
#pragma unroll
  for (int r = 0; r < ROUNDS; ++r) {                  // all destination loads in flight at once
    const int64_t i = c0 + r * 32 + lane;
    bins[r] = i < S.cap ? dest[i] : -1;
  }
  for (int q = tid; q < NW * kHist; q += kScatterThreads) (&s_wc[0][0])[q] = 0;
  // gather fallback this step / capacity exceeded (err set by the scan): no stores /
  // no particle / no local destination in this tile (uniform tests)
  const int dmin = tmeta.x;
  if (w2 || tot > S.cap || i_begin >= n || dmin == INT32_MAX) {
    if constexpr (kStage) { __syncthreads(); mbar_wait(&s_bar, 0u); }   // the copies land in this CTA's memory: wait for them
    return;
  }
  const int tcnt = (int)min((int64_t)TILE, n - i_begin);
  if constexpr (kStage) {
    const int k = tbulk / (int)sizeof(Real) + tid;     // a ragged tail (capacity not a multiple of 4), per element
    if (k < tcnt) { st_x[k] = x[i_begin + k]; st_vx[k] = vx[i_begin + k]; st_vy[k] = vy[i_begin + k]; st_vz[k] = vz[i_begin + k]; }
  }
  // ---- pass 1: this warp's destinations (kept in registers) and bin counts ----
  __syncthreads();
  if (tid < kHist) s_off[tid] = dmin + tid <= S.C ? off_new[dmin + tid] : 0;
#pragma unroll
  for (int r = 0; r < ROUNDS; ++r) {
    const int d = bins[r];
    const bool loc = c0 + r * 32 + lane < n && d >= 0 && d < S.C && d - dmin < kHist;
    bins[r] = loc ? d - dmin : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, loc ? bins[r] : -1 - lane);
    if (loc && __ffs(peers) - 1 == lane) s_wc[warp][bins[r]] += __popc(peers);
    __syncwarp();
  }
  // ---- prefix per bin: lcnt + look-back over earlier tiles, 32 at a time ----
  const int b = tid & (kHist - 1), part = tid / kHist;
  int acc = 0;
  for (int t0 = t - 1;; t0 -= 32) {
    if (warp == 0) {
      const int tp = t0 - lane;
      int2 m = make_int2(INT32_MAX, -1);
      bool stop = tp < 0;
      if (!stop) { m = t0 == t - 1 ? mprev : tile_meta[tp]; stop = m.y + Wd < dmin; }
      const unsigned st = __ballot_sync(0xffffffffu, stop);
      const int nb = st ? __ffs(st) - 1 : 32;
      s_meta[lane] = m;
      if (lane == 0) { s_nb = nb; s_more = st == 0u; }
    }
    __syncthreads();
    const int nb = s_nb;
    for (int j = part; j < nb; j += PARTS) {
      const int2 m = s_meta[j];
      const int bb = dmin + b - m.x;
      if (m.x != INT32_MAX && bb >= 0 && bb < kHist) acc += tileH[(size_t)(t0 - j) * kHist + bb];
    }
    const int more = s_more;
    __syncthreads();
    if (!more) break;
  }
  s_part[part][b] = acc;
  __syncthreads();
  if (tid < kHist) {
    int p = 0;
#pragma unroll
    for (int q = 0; q < PARTS; ++q) p += s_part[q][tid];
    const int d = dmin + tid;
    if (d < kEdgeBins && d < S.C) p += lcnt[d];
    // running start of each warp's chunk in this bin (exclusive prefix over warps)
    for (int w = 0; w < NW; ++w) { const int cw = s_wc[w][tid]; s_wc[w][tid] = p; p += cw; }
  }
  __syncthreads();
  // ---- pass 2: stable positions, in index order within the warp's chunk ----
  int rk[ROUNDS];
#pragma unroll
  for (int r = 0; r < ROUNDS; ++r) {
    const int bin = bins[r];
    const unsigned peers = __match_any_sync(0xffffffffu, bin >= 0 ? bin : -1 - lane);
    rk[r] = 0;
    if (bin >= 0) rk[r] = s_wc[warp][bin] + __popc(peers & ((1u << lane) - 1u));
    __syncwarp();
    if (bin >= 0 && __ffs(peers) - 1 == lane) s_wc[warp][bin] += __popc(peers);
    __syncwarp();
  }
  if constexpr (kStage) {
    mbar_wait(&s_bar, 0u);
    __syncthreads();                                  // the tail's generic writes
#pragma unroll
    for (int r = 0; r < ROUNDS; ++r) {
      const int bin = bins[r];
      if (bin >= 0) {
        const int k = warp * CHUNK + r * 32 + lane;
        const int64_t pos = s_off[bin] + rk[r];
        if (pos < S.cap) {
          const Real vxk = st_vx[k];
          ox[pos] = moved_x<Real>(S, st_x[k], vxk); ovx[pos] = vxk; ovy[pos] = st_vy[k]; ovz[pos] = st_vz[k];
        }
      }
    }
    pdl_trigger();
    return;
  }
  // ---- data movement: independent 4-round batches of loads, then the stores ----
  constexpr int BATCH = ROUNDS < 4 ? ROUNDS : 4;
#pragma unroll
  for (int r0 = 0; r0 < ROUNDS; r0 += BATCH) {
    Real a[BATCH], bx[BATCH], by[BATCH], bz[BATCH];
#pragma unroll
    for (int q = 0; q < BATCH; ++q) {
      const int64_t i = c0 + (r0 + q) * 32 + lane;
      if (bins[r0 + q] >= 0) { a[q] = x[i]; bx[q] = vx[i]; by[q] = vy[i]; bz[q] = vz[i]; }
    }
#pragma unroll
    for (int q = 0; q < BATCH; ++q) {
      const int bin = bins[r0 + q];
      if (bin >= 0) {
        const int64_t pos = s_off[bin] + rk[r0 + q];
        if (pos < S.cap) {
          ox[pos] = moved_x<Real>(S, a[q], bx[q]); ovx[pos] = bx[q]; ovy[pos] = by[q]; ovz[pos] = bz[q];
        }
      }
    }
  }
  pdl_trigger();
}

struct GatherSrc {
  const int64_t *off_old;
  const int *ng;
  const int *W;
  const void *recv[2];                // immigrants from the left / right neighbour (or null)
  int xcap;
  int cbase;
  const void *x, *vx, *vy, *vz;      // interior (source buffer, transported positions)
  const int32_t *dest;
  const void *gx[2], *gvx[2], *gvy[2], *gvz[2];
  const int32_t *gdest[2];
  int scatter;                        // 1: scatter_sorted placed the particles (unless W[2] is set)
};

// Stable gather of destination cell c into (bx,by,bz) [velocities] and ox
// [positions, global] in canonical source order.  Returns the count.
// Each round covers blockDim*8 source entries: a thread tests 8 consecutive
// destinations (independent loads in flight), a CTA exclusive scan of the
// per-thread match counts gives every match its stable position.
template <typename Real>
__device__ int gather_cell(const ShockDev &S, const GatherSrc &G, int c, Real *bx, Real *by, Real *bz,
                           Real *ox, int *wcnt) {
  constexpr int R = 8;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int W = *G.W;
  int running = 0;
  // canonical source order: left reservoir ghosts, left immigrants, interior,
  // right immigrants, right reservoir ghosts
  for (int seg = 0; seg < 5; ++seg) {
    int64_t lo = 0, hi = 0;
    const Real *sx, *svx, *svy, *svz;
    const int32_t *sd;
    int match = c;                       // destination value to look for
    if (seg == 2) {
      const int a = max(c - W, 0), b = min(c + W, S.C - 1);
      lo = G.off_old[a]; hi = G.off_old[b + 1];
      sx = (const Real *)G.x; svx = (const Real *)G.vx; svy = (const Real *)G.vy; svz = (const Real *)G.vz;
      sd = G.dest;
    } else if (seg == 1 || seg == 3) {
      const int side = seg == 1 ? 0 : 1;
      const bool in = side == 0 ? (c - W <= -1) : (c + W >= S.C);
      if (!in || G.recv[side] == nullptr) continue;
      const XBuf<Real> X = XBuf<Real>::bind(const_cast<void *>(G.recv[side]), G.xcap);
      hi = min(*X.count, G.xcap);
      sx = X.x; svx = X.vx; svy = X.vy; svz = X.vz; sd = X.dest;
      match = c + G.cbase;               // immigrants carry global destinations
    } else {
      const int side = seg == 0 ? 0 : 1;
      const bool in = side == 0 ? (c - W <= -1) : (c + W >= S.C);
      if (!in) continue;
      hi = G.ng[side];
      sx = (const Real *)G.gx[side]; svx = (const Real *)G.gvx[side];
      svy = (const Real *)G.gvy[side]; svz = (const Real *)G.gvz[side];
      sd = G.gdest[side];
    }
    for (int64_t b0 = lo; b0 < hi; b0 += (int64_t)blockDim.x * R) {
      const int64_t i0 = b0 + (int64_t)tid * R;
      unsigned bits = 0;
#pragma unroll
      for (int k = 0; k < R; ++k) {
        const int64_t i = i0 + k;
        if (i < hi && sd[i] == match) bits |= 1u << k;
      }
      const int mine = __popc(bits);
      int incl = mine;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      if (lane == 31) wcnt[warp] = incl;
      __syncthreads();
      int wb = 0, tot = 0;
      for (int w = 0; w < nw; ++w) {
        const int t = wcnt[w];
        wb += (w < warp) ? t : 0;
        tot += t;
      }
      const int pos = running + wb + incl - mine;
      // all loads of this thread's matches first (independent, in flight), then the stores
      Real tx[R], tvx[R], tvy[R], tvz[R];
#pragma unroll
      for (int k = 0; k < R; ++k) {
        if ((bits >> k) & 1u) {
          const int64_t i = i0 + k;
          tx[k] = sx[i]; tvx[k] = svx[i]; tvy[k] = svy[i]; tvz[k] = svz[i];
          if (seg == 2) tx[k] = moved_x<Real>(S, tx[k], tvx[k]);
        }
      }
#pragma unroll
      for (int k = 0; k < R; ++k) {
        if ((bits >> k) & 1u) {
          const int q = pos + __popc(bits & ((1u << k) - 1u));
          bx[q] = tvx[k]; by[q] = tvy[k]; bz[q] = tvz[k]; ox[q] = tx[k];
        }
      }
      running += tot;
      __syncthreads();
    }
  }
  return running;
}

// Warp-level stable gather of destination cell c (same canonical order as
// gather_cell): each lane tests 8 consecutive source entries per round, a warp
// scan gives the positions.  Velocities -> (bx,by,bz) (the warp's slab),
// positions -> ox (global).  Returns the count; sums of the velocities in s*.
template <typename Real>
__device__ __noinline__ int gather_cell_warp(const ShockDev &S, const GatherSrc &G, int c, Real *bx, Real *by, Real *bz,
                                Real *ox, int cap, double &sxo, double &syo, double &szo) {
  constexpr int R = 4;
  const int lane = threadIdx.x & 31;
  const int W = *G.W;
  int running = 0;
  double sx = 0, sy = 0, sz = 0;
  for (int seg = 0; seg < 5; ++seg) {
    int64_t lo = 0, hi = 0;
    const Real *px, *pvx, *pvy, *pvz;
    const int32_t *pd;
    int match = c;
    if (seg == 2) {
      const int a = max(c - W, 0), b = min(c + W, S.C - 1);
      lo = G.off_old[a]; hi = G.off_old[b + 1];
      px = (const Real *)G.x; pvx = (const Real *)G.vx; pvy = (const Real *)G.vy; pvz = (const Real *)G.vz;
      pd = G.dest;
    } else if (seg == 1 || seg == 3) {
      const int side = seg == 1 ? 0 : 1;
      const bool in = side == 0 ? (c - W <= -1) : (c + W >= S.C);
      if (!in || G.recv[side] == nullptr) continue;
      const XBuf<Real> X = XBuf<Real>::bind(const_cast<void *>(G.recv[side]), G.xcap);
      hi = min(*X.count, G.xcap);
      px = X.x; pvx = X.vx; pvy = X.vy; pvz = X.vz; pd = X.dest;
      match = c + G.cbase;
    } else {
      const int side = seg == 0 ? 0 : 1;
      const bool in = side == 0 ? (c - W <= -1) : (c + W >= S.C);
      if (!in) continue;
      hi = G.ng[side];
      px = (const Real *)G.gx[side]; pvx = (const Real *)G.gvx[side];
      pvy = (const Real *)G.gvy[side]; pvz = (const Real *)G.gvz[side];
      pd = G.gdest[side];
    }
    for (int64_t b0 = lo; b0 < hi; b0 += 32 * R) {
      const int64_t i0 = b0 + (int64_t)lane * R;
      unsigned bits = 0;
#pragma unroll
      for (int k = 0; k < R; ++k) {
        const int64_t i = i0 + k;
        if (i < hi && pd[i] == match) bits |= 1u << k;
      }
      const int mine = __popc(bits);
      int incl = mine;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      const int tot = __shfl_sync(0xffffffffu, incl, 31);
      const int pos = running + incl - mine;
      Real tx[R], tvx[R], tvy[R], tvz[R];
#pragma unroll
      for (int k = 0; k < R; ++k) {
        if ((bits >> k) & 1u) {
          const int64_t i = i0 + k;
          tx[k] = px[i]; tvx[k] = pvx[i]; tvy[k] = pvy[i]; tvz[k] = pvz[i];
          if (seg == 2) tx[k] = moved_x<Real>(S, tx[k], tvx[k]);
        }
      }
#pragma unroll
      for (int k = 0; k < R; ++k) {
        if ((bits >> k) & 1u) {
          const int q = pos + __popc(bits & ((1u << k) - 1u));
          if (q < cap) { bx[q] = tvx[k]; by[q] = tvy[k]; bz[q] = tvz[k]; }
          ox[q] = tx[k];
          sx += tvx[k]; sy += tvy[k]; sz += tvz[k];
        }
      }
      running += tot;
    }
  }
  sxo = sx; syo = sy; szo = sz;
  __syncwarp();
  return running;
}

template <typename Real, bool WB>
__global__ void __launch_bounds__(kWarpCellWarps * 32, TRMCR_WARP_MINB)
shock_collide_warp(StepParams P, WarpSlabLayout Lay, ShockDev S, GatherSrc G, const int64_t *__restrict__ off_new,
                   Real *ox, Real *ovx, Real *ovy, Real *ovz, int32_t *m_state, double *stats, int *defer_count,
                   int *defer_list, QueueArgs Q) {
  pdl_wait();   // programmatic dependent launch: the predecessor's writes are visible
  if (off_new[S.C] > S.cap) { pdl_trigger(); return; }   // capacity exceeded (err set by the scan): no stores
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char *slab = smem + (size_t)warp * Lay.per_warp;
  WarpShared &sh = *reinterpret_cast<WarpShared *>(slab + Lay.off_sh);
  CellBuf<Real> B;
  double *usplit;
  bind_warp_slab(B, slab, Lay, usplit);
  const int nw = gridDim.x * (blockDim.x >> 5);
  const bool sorted = G.scatter && !Lay.v_smem && G.W[2] == 0;
  for (int c = blockIdx.x * (blockDim.x >> 5) + warp; c < S.C; c += nw) {
    const int64_t base = off_new[c];
    const int n = (int)(off_new[c + 1] - base);
    int rc = kOverflow;
    if (n <= Lay.n_cap) {
      double sx, sy, sz;
      if (!Lay.v_smem) { B.vx = ovx + base; B.vy = ovy + base; B.vz = ovz + base; }   // work in place (L1)
      if (sorted) {                        // already in place: sums of the cell
        sx = 0; sy = 0; sz = 0;
        for (int i = lane; i < n; i += 32) { sx += B.vx[i]; sy += B.vy[i]; sz += B.vz[i]; }
      } else {
        gather_cell_warp<Real>(S, G, c, B.vx, B.vy, B.vz, ox + base, Lay.n_cap, sx, sy, sz);
      }
      if (n == 0) {
        if (lane == 0) {
          double *s = stats + (size_t)c * TRMCR_NSTATS;
          for (int k = 0; k < TRMCR_NSTATS; ++k) s[k] = 0.0;
          const int m = P.adaptive ? m_state[c] : P.m_fixed;
          s[TRMCR_ST_MUSED] = m; s[TRMCR_ST_MNEXT] = m;
        }
        rc = kOk;
      } else {
        rc = process_cell_warp<Real, WB>(P, B, sh, usplit, sx, sy, sz, ovx + base, ovy + base, ovz + base, n,
                                     P.cell_base + (uint32_t)c, m_state + c, stats + (size_t)c * TRMCR_NSTATS,
                                     Q.log, Q.log_count, Q.log_cap);
      }
    }
    if (rc != kOk && lane == 0) defer_list[atomicAdd(defer_count, 1)] = c;
    __syncwarp();
  }
  pdl_trigger();
}

// Lock-step variant of shock_collide_warp: CTAs of kLockWarps warps take
// kLockWarps neighbouring cells (similar cost) per round and run the phases of
// the general step (cell_warp.cuh: begin, attempts, end) with a CTA barrier
// between phases, so the warps of a group execute the same phase's code (the
// ~90 KB kernel body exceeds the 32 KB instruction cache; free-running warps
// stall on instruction fetch: 5.3 cycles per issue, 0.2 in lock step).  Small
// groups bound the barrier idle of unequal cells.  Sorted cells only (no
// gather); results identical to the free-running kernel.
// Group size x CTAs per SM, measured on C5 (collision kernel, ms; the register
// cap follows from the launch bounds, none of these spills):
//   round 1 (another kernel body): 16x1 2.02, 8x2 1.80, 4x4 1.66, 2x8 +0.09, free-running 1.75
//   round 2: 4x4 (116 regs) 1.233, 8x2 (116) 1.211, 16x1 1.282, 3x5 1.344, 5x3 1.253, 6x3 (96) 1.232,
//            7x2 1.327, 9x2 (96) 1.242, 10x2 (96 regs, 20 warps per SM) 1.155, 5x4 (96) 1.250,
//            4x5 (96) 1.322, 20x1 (96) 1.250, 12x1 1.486, 7x3 / 11x2 / 12x2 (80 regs, spills) 1.26 / 1.25 / 1.20
#ifndef TRMCR_LOCK_WARPS
#define TRMCR_LOCK_WARPS 10
#endif
constexpr int kLockWarps = TRMCR_LOCK_WARPS;
#ifndef TRMCR_LOCK_MINB
#define TRMCR_LOCK_MINB (20 / TRMCR_LOCK_WARPS)
#endif
// TRMCR_LOCK_GROUPS > 1: a CTA holds that many independent lock-step groups;
// group g = warp % groups, so the kLockWarps warps of a group have the same
// warp id modulo 4 (one SM sub-partition: its instruction cache serves one
// phase) and synchronise on their own named barrier.
#ifndef TRMCR_LOCK_GROUPS
#define TRMCR_LOCK_GROUPS 1
#endif
constexpr int kLockGroups = TRMCR_LOCK_GROUPS;
constexpr int kLockThreads = kLockWarps * kLockGroups * 32;
__device__ __forceinline__ void lock_group_barrier(int grp) {
  if constexpr (kLockGroups == 1) __syncthreads();
  else asm volatile("bar.sync %0, %1;" ::"r"(grp + 1), "n"(kLockWarps * 32) : "memory");
}
template <typename Real, bool WB, int MOD = -1>
__global__ void __launch_bounds__(kLockThreads, (TRMCR_LOCK_MINB + kLockGroups - 1) / kLockGroups)
shock_collide_lock(StepParams P, WarpSlabLayout Lay, ShockDev S, GatherSrc G, const int64_t *__restrict__ off_new,
                   Real *ox, Real *ovx, Real *ovy, Real *ovz, int32_t *m_state, double *stats, int *defer_count,
                   int *defer_list, QueueArgs Q) {
  pdl_wait();   // programmatic dependent launch: the predecessor's writes are visible
  if (off_new[S.C] > S.cap) { pdl_trigger(); return; }   // capacity exceeded (err set by the scan): no stores
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char *slab = smem + (size_t)warp * Lay.per_warp;
  WarpShared &sh = *reinterpret_cast<WarpShared *>(slab + Lay.off_sh);
  CellBuf<Real> B;
  double *usplit;
  bind_warp_slab(B, slab, Lay, usplit);
  const int grp = warp % kLockGroups, mem = warp / kLockGroups;
  for (int base = (blockIdx.x * kLockGroups + grp) * kLockWarps; base < S.C;
       base += gridDim.x * kLockGroups * kLockWarps) {
    const int c = base + mem;
    int64_t b0 = 0;
    int n = 0, rc = kOk;
    bool run = false;                         // this warp's cell still has phases to run
#ifdef TRMCR_LOCK_PREFETCH
    int64_t nb = 0;                           // this warp's next cell: its offsets come with this cell's
    int nn = 0;
    if (c + (int)(gridDim.x * kLockGroups * kLockWarps) < S.C) {
      const int cn = c + (int)(gridDim.x * kLockGroups * kLockWarps);
      nb = off_new[cn];
      nn = (int)(off_new[cn + 1] - nb);
    }
#endif
    if (c < S.C) {
      b0 = off_new[c];
      n = (int)(off_new[c + 1] - b0);
      B.vx = ovx + b0; B.vy = ovy + b0; B.vz = ovz + b0;
      if (n > Lay.n_cap) {
        rc = kOverflow;
      } else if (n == 0) {
        if (lane == 0) {
          double *st = stats + (size_t)c * TRMCR_NSTATS;
          for (int k = 0; k < TRMCR_NSTATS; ++k) st[k] = 0.0;
          const int m = P.adaptive ? m_state[c] : P.m_fixed;
          st[TRMCR_ST_MUSED] = m; st[TRMCR_ST_MNEXT] = m;
        }
      } else {
        PHASE_MARK(t_b);
        double sx = 0, sy = 0, sz = 0;
        if constexpr (sizeof(Real) == 4) {
          warp_cell_sums(B.vx, B.vy, B.vz, n, sx, sy, sz);
        } else {
          for (int i = lane; i < n; i += 32) { sx += B.vx[i]; sy += B.vy[i]; sz += B.vz[i]; }
        }
        WPHASE_ADD(9, t_b);   // load sums
        rc = wphase_begin<Real, MOD>(P, B, sh, usplit, sx, sy, sz, n, P.cell_base + (uint32_t)c, m_state + c);
        WPHASE_ADD(0, t_b);   // moments + split
        run = rc == kOk;
      }
    }
#ifdef TRMCR_LOCK_PREFETCH
    if (nn > 0 && lane < 3) {                 // the next cell's velocities into L2 while this one collides
      const Real *p = (lane == 0 ? ovx : lane == 1 ? ovy : ovz) + nb;
      const uintptr_t a = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15);
      prefetch_l2(reinterpret_cast<const void *>(a),
                  (unsigned)((reinterpret_cast<uintptr_t>(p + nn) + 15 - a) & ~uintptr_t(15)));
    }
#endif
    const bool work = run;
    PHASE_MARK(t_w);
    // the begin phase ends in lock step; the attempts (attempt 0 and any RAD
    // retries) run free - a barrier per attempt measured slower (C5 1.61 vs
    // 1.53 ms: retries are a minority of the cells)
#ifndef TRMCR_LOCK_NO_BEGIN_BARRIER
    lock_group_barrier(grp);
#endif
    WPHASE_ADD(10, t_w);   // barrier after begin
#ifdef TRMCR_LOCK_ATTEMPT_SYNC
    // every attempt in lock step too: the group iterates until none of its cells retries
    static_assert(kLockGroups == 1, "the vote is CTA wide");
    while (__syncthreads_or(run ? 1 : 0)) {
      if (run) {
        rc = wphase_attempt<Real, WB, MOD>(P, B, sh, usplit, P.cell_base + (uint32_t)c, Q.log, Q.log_count, Q.log_cap);
        run = rc == kOk && !sh.done;
      }
    }
#else
    while (run) {
      rc = wphase_attempt<Real, WB, MOD>(P, B, sh, usplit, P.cell_base + (uint32_t)c, Q.log, Q.log_count, Q.log_cap);
      run = rc == kOk && !sh.done;
    }
#endif
    PHASE_MARK(t_e);
    if (work && rc == kOk)
      wphase_end<Real, WB>(P, B, sh, B.vx, B.vy, B.vz, P.cell_base + (uint32_t)c, m_state + c,
                       stats + (size_t)c * TRMCR_NSTATS);
    WPHASE_ADD(6, t_e);   // Maxwellian + stats
    if (c < S.C && rc != kOk && lane == 0) defer_list[atomicAdd(defer_count, 1)] = c;
#ifndef TRMCR_LOCK_NO_END_BARRIER
    lock_group_barrier(grp);                          // round in lock step (dropping it measured slower)
#endif
    WPHASE_ADD(11, t_e);   // barrier at round end
  }
  pdl_trigger();
}

}  // namespace trmcr
#include "fused.cuh"
namespace trmcr {

template <typename Real, int THREADS>
__global__ void __launch_bounds__(THREADS, 768 / THREADS)
shock_collide_smem(StepParams P, SmemLayout Lay, ShockDev S, GatherSrc G, FusedDev F, int par_in, int fused,
                   const int64_t *__restrict__ off_new,
                   Real *ox, Real *ovx, Real *ovy, Real *ovz, int32_t *m_state, double *stats,
                   const int *list_count, const int *list, QueueArgs Q) {
  pdl_wait();   // programmatic dependent launch: the predecessor's writes are visible
  if (off_new[S.C] > S.cap) { pdl_trigger(); return; }   // capacity exceeded (err set by the scan): no stores
  BlockTeam team;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ CellShared sh;
  __shared__ int wcnt[32];
  const int count = list ? *list_count : S.C;
  CellBuf<Real> B;
  bind_smem(B, smem, Lay);
  for (int k = blockIdx.x; k < count; k += gridDim.x) {
  const int c = list ? list[k] : k;
  const int64_t base = off_new[c];
  const int n = (int)(off_new[c + 1] - base);
  int rc = kOverflow;
  if (n <= B.n_cap) {
    PHASE_MARK(t_g);
    if (fused) {   // re-place the cell from the source (the fused pass may have left it half-stepped)
      if (threadIdx.x < 32)
        gather_fused_warp<Real>(S, G, F, par_in, c, ox + base, ovx + base, ovy + base, ovz + base, n);
      __syncthreads();
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        B.vx[i] = ovx[base + i]; B.vy[i] = ovy[base + i]; B.vz[i] = ovz[base + i];
      }
    } else {
      gather_cell<Real>(S, G, c, B.vx, B.vy, B.vz, ox + base, wcnt);
    }
    __syncthreads();
    PHASE_ADD(8, t_g);   // gather
    rc = process_cell<Real, false, true>(team, P, B, sh, nullptr, nullptr, nullptr, ovx + base, ovy + base,
                                         ovz + base, n, P.cell_base + (uint32_t)c, m_state + c,
                                         stats + (size_t)c * TRMCR_NSTATS, Q.log, Q.log_count, Q.log_cap);
    if (fused && rc == kOk) {
      __syncthreads();
      if (threadIdx.x < 32) warp_codes<Real>(S, F, par_in ^ 1, c, base, n, ox, ovx, Q.err);
    }
  }
  if (rc != kOk && threadIdx.x == 0) {
    const int j = atomicAdd(Q.ovf_count, 1);
    Q.ovf_list[j] = c;
  }
  __syncthreads();
  }
  pdl_trigger();
}

template <typename Real>
__global__ void __launch_bounds__(kGmemThreads)
shock_collide_gmem(StepParams P, GmemScratch GS, ShockDev S, GatherSrc G, FusedDev F, int par_in, int fused,
                   const int64_t *__restrict__ off_new,
                   Real *ox, Real *ovx, Real *ovy, Real *ovz, int32_t *m_state, double *stats, QueueArgs Q) {
  pdl_wait();   // programmatic dependent launch: the predecessor's writes are visible
  if (off_new[S.C] > S.cap) { pdl_trigger(); return; }   // capacity exceeded (err set by the scan): no stores
  BlockTeam team;
  __shared__ CellShared sh;
  __shared__ double red[32 * 8];
  __shared__ int wcnt[32];
  const int count = *Q.ovf_count;
  CellBuf<Real> B;
  bind_gmem(B, GS, red);
  for (int k = blockIdx.x; k < count; k += gridDim.x) {
    const int c = Q.ovf_list[k];
    const int64_t base = off_new[c];
    const int n = (int)(off_new[c + 1] - base);
    B.vx = ovx + base; B.vy = ovy + base; B.vz = ovz + base;
    if (fused) {
      if (threadIdx.x < 32)
        gather_fused_warp<Real>(S, G, F, par_in, c, ox + base, ovx + base, ovy + base, ovz + base, n);
    } else {
      gather_cell<Real>(S, G, c, B.vx, B.vy, B.vz, ox + base, wcnt);
    }
    __syncthreads();
    const int rc = process_cell<Real, false, false>(team, P, B, sh, nullptr, nullptr, nullptr, B.vx, B.vy, B.vz, n,
                                                    P.cell_base + (uint32_t)c, m_state + c,
                                                    stats + (size_t)c * TRMCR_NSTATS, Q.log, Q.log_count,
                                                    Q.log_cap);
    if (rc != kOk && threadIdx.x == 0) atomicOr(Q.err, 1);
    if (fused && rc == kOk) {
      __syncthreads();
      if (threadIdx.x < 32) warp_codes<Real>(S, F, par_in ^ 1, c, base, n, ox, ovx, Q.err);
    }
    __syncthreads();
  }
  pdl_trigger();
}

inline FusedDev fused_dev(const trmcr_ctx *c) {
  const ShockState &s = c->shock;
  FusedDev f;
  for (int k = 0; k < 2; ++k) {
    f.code[k] = s.d_code[k]; f.nlsr[k] = s.d_nlsr[k]; f.far_src[k] = s.d_far_src[k]; f.far_dst[k] = s.d_far_dst[k];
  }
  f.far_cnt = s.d_far_cnt;
  f.far_cap = s.far_cap;
  return f;
}

inline ShockDev shock_dev(const trmcr_ctx *c) {
  const ShockState &s = c->shock;
  ShockDev d;
  d.C = s.C; d.Cg = s.Cg; d.cbase = s.cbase; d.has_left = s.has_left; d.has_right = s.has_right;
  d.x_min = s.x_min; d.x_max = s.x_max; d.inv_dx = s.inv_dx; d.dt = c->dt;
  auto ceil_f = [](double v) { float f = (float)v; return (double)f < v ? nextafterf(f, INFINITY) : f; };
  d.x_min_f = ceil_f(s.x_min); d.x_max_f = ceil_f(s.x_max);
  for (int k = 0; k < 2; ++k) {
    d.rho[k] = s.rho[k]; d.u[k] = s.u[k]; d.T[k] = s.T[k]; d.Lg[k] = s.Lg[k];
    d.y[k] = s.rho[k] * s.Lg[k] / s.weight;
  }
  d.cap_g = s.cap_g;
  d.cap = c->cap;
  d.n_hint = c->n - c->n / 16;
  return d;
}

inline trmcr_status shock_rebin(trmcr_ctx *c, int *max_cell);

// Allocate shock state, validate + count the initial particles (inside this
// slab, sorted by cell), build offsets.  Synchronises (init only).
inline trmcr_status shock_init(trmcr_ctx *c, const trmcr_cells *cc, int *max_cell) {
  ShockState &s = c->shock;
  s.C = cc->n_cells;
  s.Cg = cc->n_cells_global > 0 ? cc->n_cells_global : cc->n_cells;
  s.cbase = cc->cell_base;
  s.has_left = (cc->neighbors & 1) ? 1 : 0;
  s.has_right = (cc->neighbors & 2) ? 1 : 0;
  if (s.cbase + s.C > s.Cg) return fail(c, TRMCR_EINVAL, "slab outside the global grid");
  if (s.has_left != (s.cbase > 0) || s.has_right != (s.cbase + s.C < s.Cg))
    return fail(c, TRMCR_EINVAL, "neighbours must be exactly the slabs next to this one");
  s.x_min = cc->x_min; s.x_max = cc->x_max; s.weight = cc->weight;
  s.inv_dx = (double)s.Cg / (cc->x_max - cc->x_min);
  s.rho[0] = cc->rho_L; s.u[0] = cc->u_L; s.T[0] = cc->T_L;
  s.rho[1] = cc->rho_R; s.u[1] = cc->u_R; s.T[1] = cc->T_R;
  double ymax = 0;
  for (int k = 0; k < 2; ++k) {
    s.Lg[k] = (fabs(s.u[k]) + 6.0 * sqrt(s.T[k])) * c->dt;
    ymax = std::max(ymax, s.rho[k] * s.Lg[k] / s.weight);
  }
  if (ymax > 1e9) return fail(c, TRMCR_EINVAL, "reservoir ghost slab too large (dt / weight)");
  s.cap_g = (int)floor(ymax) + 2;   // IR(y) <= floor(y) + 1
  if (dalloc(c, &s.d_off[0], sizeof(int64_t) * (s.C + 1)) || dalloc(c, &s.d_off[1], sizeof(int64_t) * (s.C + 1)) ||
      dalloc(c, &s.d_dest, sizeof(int32_t) * (size_t)c->cap) || dalloc(c, &s.d_counts, sizeof(int32_t) * s.C) ||
      dalloc(c, &s.d_ng, sizeof(int) * 2) || dalloc(c, &s.d_W, sizeof(int) * 3) ||
      dalloc(c, &s.d_acct, sizeof(unsigned long long) * 4))
    return TRMCR_ENOMEM;
  for (int k = 0; k < 2; ++k) {
    if (dalloc(c, &s.d_gdest[k], sizeof(int32_t) * s.cap_g) || dalloc(c, &s.gx[k], c->rs * s.cap_g)) return TRMCR_ENOMEM;
    for (int j = 0; j < 3; ++j)
      if (dalloc(c, &s.gv[k][j], c->rs * s.cap_g)) return TRMCR_ENOMEM;
  }
  if (const char *se = getenv("TRMCR_SHOCK_SCATTER")) s.scatter = atoi(se) != 0;
  // transport / sort tiles: 1024 x TRMCR_TILE_GROUPS (2048) particles for large problems, 1024 below 8 M
  // particles (more CTAs in flight: C4 has 1 M)
  s.tile_ng = c->cap >= (int64_t)8 << 20 ? kTransportGroups : 1;
  if (const char *te = getenv("TRMCR_TILE_NG")) s.tile_ng = atoi(te) == 1 ? 1 : kTransportGroups;
  s.ntiles = (int)((c->cap + tile_of(s.tile_ng) - 1) / tile_of(s.tile_ng));
  if (s.scatter && (dalloc(c, &s.d_tileH, sizeof(int32_t) * kHist * (size_t)std::max(s.ntiles, 1)) ||
                    dalloc(c, &s.d_tile_meta, sizeof(int2) * (size_t)std::max(s.ntiles, 1)) ||
                    dalloc(c, &s.d_lcnt, sizeof(int32_t) * kEdgeBins)))
    return TRMCR_ENOMEM;
  const int scan_blocks = std::max(1, (s.C + kScanTile - 1) / kScanTile);
  {   // decoupled look-back needs every scan CTA resident at once (spin-waits on predecessors)
    int nsm = 148, occ = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, scan_offsets_lb, kScanThreads, 0) != cudaSuccess) {
      cudaGetLastError();
      occ = 0;
    }
    s.scan_lb = scan_blocks <= nsm * occ / 2;
  }
  if (dalloc(c, &s.d_scan_status, sizeof(unsigned long long) * scan_blocks)) return TRMCR_ENOMEM;
  CUDA_TRY(c, cudaMemsetAsync(s.d_scan_status, 0, sizeof(unsigned long long) * scan_blocks, c->stream));
  s.scan_epoch = 0;
  CUDA_TRY(c, cudaMemsetAsync(s.d_acct, 0, sizeof(unsigned long long) * 4, c->stream));
  CUDA_TRY(c, cudaMemsetAsync(s.d_ng, 0, sizeof(int) * 2, c->stream));
  c->cur = 0;
  return shock_rebin(c, max_cell);
}

// Bin the c->n particles of buffer c->cur (positions inside this slab, sorted by
// cell: validated) into d_off[cur]; *max_cell = the largest cell.  Used by init
// and by trmcr_set_particles.  Synchronises.  EINVAL (not sticky) on bad input.
inline trmcr_status shock_rebin(trmcr_ctx *c, int *max_cell) {
  ShockState &s = c->shock;
  const int cur = c->cur;
  s.codes_ok = 0;
  CUDA_TRY(c, cudaMemsetAsync(s.d_counts, 0, sizeof(int32_t) * s.C, c->stream));
  const ShockDev d = shock_dev(c);
  if (c->n > 0) {
    const unsigned blocks = (unsigned)((c->n + 255) / 256);
    if (c->dtype == TRMCR_F64)
      shock_bin_init<double><<<blocks, 256, 0, c->stream>>>(d, (const double *)c->x[cur], c->n, s.d_counts, c->d_err);
    else
      shock_bin_init<float><<<blocks, 256, 0, c->stream>>>(d, (const float *)c->x[cur], c->n, s.d_counts, c->d_err);
    if (auto e = check_launch(c, "shock_bin_init")) return e;
  }
  scan_offsets<<<1, 1024, 0, c->stream>>>(s.d_counts, s.C, s.d_off[cur], c->cap, c->d_err);
  if (auto e = check_launch(c, "scan_offsets")) return e;
  std::vector<int32_t> counts(s.C);
  CUDA_TRY(c, cudaMemcpyAsync(counts.data(), s.d_counts, sizeof(int32_t) * s.C, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  int err = 0;
  CUDA_TRY(c, cudaMemcpy(&err, c->d_err, sizeof(int), cudaMemcpyDeviceToHost));
  c->d_offsets = s.d_off[cur];
  if (err & 12) {                          // input errors: cleared, the call fails, the context stays usable
    const int rest = err & ~12;
    CUDA_TRY(c, cudaMemcpy(c->d_err, &rest, sizeof(int), cudaMemcpyHostToDevice));
    c->n = 0;                                // no valid state until the next successful set
    CUDA_TRY(c, cudaMemsetAsync(s.d_off[cur], 0, sizeof(int64_t) * (s.C + 1), c->stream));
    if (err & 4) return fail(c, TRMCR_EINVAL, "particle outside this slab of the shock domain");
    return fail(c, TRMCR_EINVAL, "shock particles must be sorted by cell (stable order)");
  }
  if (max_cell) {
    *max_cell = 0;
    for (int32_t v : counts) *max_cell = std::max(*max_cell, (int)v);
  }
  return TRMCR_OK;
}

// Sources of the current step's gathers (buffer cur, ghosts, immigrants).
inline GatherSrc gather_src(const trmcr_ctx *c) {
  const ShockState &s = c->shock;
  const int cur = c->cur;
  GatherSrc G;
  G.off_old = s.d_off[cur]; G.ng = s.d_ng; G.W = s.d_W;
  G.x = c->x[cur]; G.vx = c->v[cur][0]; G.vy = c->v[cur][1]; G.vz = c->v[cur][2]; G.dest = s.d_dest;
  for (int k = 0; k < 2; ++k) {
    G.gx[k] = s.gx[k]; G.gvx[k] = s.gv[k][0]; G.gvy[k] = s.gv[k][1]; G.gvz[k] = s.gv[k][2];
    G.gdest[k] = s.d_gdest[k];
  }
  G.recv[0] = s.has_left ? s.xrecv[0] : nullptr;
  G.recv[1] = s.has_right ? s.xrecv[1] : nullptr;
  G.xcap = s.xcap;
  G.cbase = s.cbase;
  G.scatter = 0;
  return G;
}

// Phase 1 of a shock step: reservoirs, transport, counts, emigrant packing.
template <typename Real>
trmcr_status shock_begin(trmcr_ctx *c) {
  ShockState &s = c->shock;
  const ShockDev d = shock_dev(c);
  const int cur = c->cur;
  prof_begin(c, TRMCR_K_GHOST_COUNT);

  launch_k(c, shock_prologue, std::max(1, std::min(32, (s.C + 4095) / 4096)), 256, (size_t)(0), d, c->P.k0, c->P.k1, c->step, s.d_ng, c->d_err, s.d_counts, s.d_W, s.d_acct, c->d_ovf_count,
      c->d_defer_count, s.fused ? s.d_far_cnt + (cur ^ 1) : (int *)nullptr);
  if (auto e = check_launch(c, "shock_prologue", TRMCR_K_GHOST_COUNT)) return e;
  if (s.fused && !s.codes_ok) {   // codes of the current state (after init / an upload)
    CUDA_TRY(c, cudaMemsetAsync(s.d_far_cnt + cur, 0, sizeof(int), c->stream));
    launch_k(c, codes_kernel<Real>, std::max(1, std::min(148 * 8, (s.C + 7) / 8)), 256, (size_t)0, d, fused_dev(c), cur,
             (const int64_t *)s.d_off[cur], (const Real *)c->x[cur], (const Real *)c->v[cur][0], c->d_err);
    if (auto e = check_launch(c, "codes_kernel")) return e;
    s.codes_ok = 1;
  }
  {
    dim3 grid((unsigned)((s.cap_g + 255) / 256), 2);
    prof_begin(c, TRMCR_K_GHOST_GEN);
    launch_k(c, ghost_gen<Real>, grid, 256, (size_t)(0), d, c->P.k0, c->P.k1, c->step, s.d_ng, (Real *)s.gx[0], (Real *)s.gx[1], (Real *)s.gv[0][0],
        (Real *)s.gv[0][1], (Real *)s.gv[0][2], (Real *)s.gv[1][0], (Real *)s.gv[1][1], (Real *)s.gv[1][2],
        s.d_gdest[0], s.d_gdest[1], s.d_counts, s.d_W, s.d_acct);
    if (auto e = check_launch(c, "ghost_gen", TRMCR_K_GHOST_GEN)) return e;
  }
  if (s.fused) {
    launch_k(c, far_count, 1, 256, (size_t)0, fused_dev(c), cur, s.d_counts, s.d_W);
    if (auto e = check_launch(c, "far_count")) return e;
    if (s.has_left || s.has_right) {
      if (!s.xsend[0] && !s.xsend[1]) return fail(c, TRMCR_EINVAL, "slab exchange buffers not set (trmcr_shock_set_exchange)");
      launch_k(c, pack_emigrants_fused<Real>, 2, 32, (size_t)0, d, gather_src(c), fused_dev(c), cur, s.xsend[0],
               s.xsend[1], s.xcap, c->d_err);
      if (auto e = check_launch(c, "pack_emigrants_fused")) return e;
    }
    return TRMCR_OK;
  }
  {
    const int per_block = tile_of(s.tile_ng);
    const unsigned blocks = (unsigned)((c->cap + per_block - 1) / per_block);
    prof_begin(c, TRMCR_K_TRANSPORT);
    const bool sc = s.scatter && c->wlay.n_cap > 0 && !c->wlay.v_smem;
    auto *tk = s.tile_ng == 1 ? transport_kernel<Real, 1> : transport_kernel<Real, kTransportGroups>;
    // a slab with neighbours: the edge tiles first (the emigrants' sources), the bulk after the pack
    launch_k(c, tk, blocks, kTransportThreads, (size_t)(0), d, s.d_off[cur], (Real *)c->x[cur], (const Real *)c->v[cur][0], s.d_dest, s.d_counts, s.d_W, s.d_acct,
        sc ? s.d_tileH : nullptr, sc ? s.d_tile_meta : nullptr, (s.has_left || s.has_right) ? 1 : 0, c->d_err);
    if (auto e = check_launch(c, "transport_kernel", TRMCR_K_TRANSPORT)) return e;
  }
  if (s.has_left || s.has_right) {
    if (!s.xsend[0] && !s.xsend[1]) return fail(c, TRMCR_EINVAL, "slab exchange buffers not set (trmcr_shock_set_exchange)");
    launch_k(c, pack_emigrants<Real>, 2, 1024, (size_t)(0), d, s.d_off[cur], s.d_ng, s.d_W, (const Real *)c->x[cur], (const Real *)c->v[cur][0],
        (const Real *)c->v[cur][1], (const Real *)c->v[cur][2], s.d_dest, (const Real *)s.gx[0],
        (const Real *)s.gv[0][0], (const Real *)s.gv[0][1], (const Real *)s.gv[0][2], s.d_gdest[0],
        (const Real *)s.gx[1], (const Real *)s.gv[1][0], (const Real *)s.gv[1][1], (const Real *)s.gv[1][2],
        s.d_gdest[1], s.xsend[0], s.xsend[1], s.xcap, c->d_err, tile_of(s.tile_ng));
    if (auto e = check_launch(c, "pack_emigrants")) return e;
    // the emigrants are packed: their exchange (comm_shock_exchange, on the
    // communication stream) overlaps the transport of the bulk
    if (c->ev_pack) CUDA_TRY(c, cudaEventRecord(c->ev_pack, c->stream));
    const int per_block = tile_of(s.tile_ng);
    const unsigned blocks = (unsigned)((c->cap + per_block - 1) / per_block);
    prof_begin(c, TRMCR_K_TRANSPORT);
    const bool sc = s.scatter && c->wlay.n_cap > 0 && !c->wlay.v_smem;
    auto *tk = s.tile_ng == 1 ? transport_kernel<Real, 1> : transport_kernel<Real, kTransportGroups>;
    launch_k(c, tk, blocks, kTransportThreads, (size_t)(0), d, s.d_off[cur], (Real *)c->x[cur], (const Real *)c->v[cur][0], s.d_dest, s.d_counts, s.d_W, s.d_acct,
        sc ? s.d_tileH : nullptr, sc ? s.d_tile_meta : nullptr, 2, c->d_err);
    if (auto e = check_launch(c, "transport_kernel", TRMCR_K_TRANSPORT)) return e;
  }
  return TRMCR_OK;
}

// Phase 2: immigrants (exchange buffers filled by the caller), offsets, the
// fused stable gather + collision step, buffer swap.
template <typename Real>
trmcr_status shock_finish(trmcr_ctx *c) {
  ShockState &s = c->shock;
  const ShockDev d = shock_dev(c);
  const int cur = c->cur, nxt = cur ^ 1;
  if (s.has_left || s.has_right) {
    dim3 grid((unsigned)((s.xcap + 255) / 256), 2);
    launch_k(c, immigrant_count<Real>, grid, 256, (size_t)(0), d, s.xrecv[0], s.xrecv[1], s.xcap, s.d_counts, s.d_W, c->d_err);
    if (auto e = check_launch(c, "immigrant_count")) return e;
  }
  if (s.fused) {
    launch_k(c, fused_counts, std::max(1, std::min(148 * 4, (s.C + 255) / 256)), 256, (size_t)0, d,
             (const int32_t *)s.d_nlsr[cur], s.d_counts);
    if (auto e = check_launch(c, "fused_counts")) return e;
  }
  prof_begin(c, TRMCR_K_SCAN);
  if (s.scan_lb)
    launch_k(c, scan_offsets_lb, std::max(1, (s.C + kScanTile - 1) / kScanTile), kScanThreads, (size_t)(0), s.d_counts, s.C, s.d_off[nxt], c->cap, c->d_err, s.d_scan_status, next_scan_epoch(s));
  else   // more scan tiles than can be resident at once: the look-back could wait on an unscheduled CTA
    launch_k(c, scan_offsets, 1, 1024, (size_t)(0), (const int32_t *)s.d_counts, s.C, s.d_off[nxt], c->cap, c->d_err);
  if (auto e = check_launch(c, "scan_offsets", TRMCR_K_SCAN)) return e;

  GatherSrc G = gather_src(c);
  QueueArgs Q{c->d_ovf_count, c->d_ovf_list, c->d_err, c->d_log, c->d_log_count, c->log_cap};
  c->P.step = c->step;
  Real *ox = (Real *)c->x[nxt], *ovx = (Real *)c->v[nxt][0], *ovy = (Real *)c->v[nxt][1], *ovz = (Real *)c->v[nxt][2];
  const bool use_warp = c->wlay.n_cap > 0;
  const FusedDev F = fused_dev(c);
  const int fz = s.fused;
  G.scatter = !fz && s.scatter && use_warp && !c->wlay.v_smem;
  if (fz) {
    prof_begin(c, TRMCR_K_SHOCK_WARP);
    const bool wb = ext_variant(c);
    launch_k(c, (wb ? shock_fused_lock<Real, true> : shock_fused_lock<Real, false>), c->lock_grid, kLockWarps * 32,
             (size_t)(c->lock_smem), c->P, c->wlay, d, G, F, cur, s.d_off[nxt], ox, ovx, ovy, ovz, c->d_mstate,
             c->d_stats, c->d_defer_count, c->d_defer_list, Q);
    if (auto e = check_launch(c, "shock_fused_lock", TRMCR_K_SHOCK_WARP)) return e;
  } else if (G.scatter) {
    prof_begin(c, TRMCR_K_SCATTER);
    launch_k(c, edge_place<Real>, 2, kEdgeThreads, (size_t)(0), d, s.d_off[nxt], s.d_ng, G.recv[0], G.recv[1], s.xcap, (const Real *)s.gx[0], (const Real *)s.gv[0][0],
        (const Real *)s.gv[0][1], (const Real *)s.gv[0][2], s.d_gdest[0], (const Real *)s.gx[1],
        (const Real *)s.gv[1][0], (const Real *)s.gv[1][1], (const Real *)s.gv[1][2], s.d_gdest[1], s.d_lcnt, ox,
        ovx, ovy, ovz, s.d_W);
    if (auto e = check_launch(c, "edge_place")) return e;
    auto *sk = s.tile_ng == 1 ? scatter_sorted<Real, 1> : scatter_sorted<Real, kTransportGroups>;
    const size_t stage = sizeof(Real) == 4 ? 4 * sizeof(Real) * (size_t)tile_of(s.tile_ng) : 0;
    launch_k(c, sk, std::max(s.ntiles, 1), kScatterThreads, stage, d, s.d_off[cur], s.d_off[nxt], (const Real *)c->x[cur], (const Real *)c->v[cur][0],
        (const Real *)c->v[cur][1], (const Real *)c->v[cur][2], s.d_dest, s.d_tileH, s.d_tile_meta, s.d_lcnt,
        s.d_W, ox, ovx, ovy, ovz);
    if (auto e = check_launch(c, "scatter_sorted", TRMCR_K_SCATTER)) return e;
  }
  if (use_warp && !fz) {
    prof_begin(c, TRMCR_K_SHOCK_WARP);
    const bool wb = ext_variant(c);
    if (G.scatter && c->batch_grid > 0)
      launch_k(c, collide_batch<Real, QueueArgs>, c->batch_grid, kBatchThreads, (size_t)c->blay.total, c->P, c->blay, s.C, c->cap,
               (const int64_t *)s.d_off[nxt], ovx, ovy, ovz, c->d_mstate, c->d_stats, c->d_defer_count,
               c->d_defer_list, Q);
    else if (G.scatter && c->lock_grid > 0)
      launch_k(c, (wb ? shock_collide_lock<Real, true>
                      : (c->P.model == TRMCR_HARD_SPHERE ? shock_collide_lock<Real, false, TRMCR_HARD_SPHERE>
                                                         : shock_collide_lock<Real, false>)), (c->lock_grid + kLockGroups - 1) / kLockGroups, kLockThreads, (size_t)(c->lock_smem) * kLockGroups, c->P, c->wlay, d, G, s.d_off[nxt], ox, ovx, ovy, ovz, c->d_mstate, c->d_stats, c->d_defer_count,
              c->d_defer_list, Q);
    else
      launch_k(c, (wb ? shock_collide_warp<Real, true> : shock_collide_warp<Real, false>), c->warp_grid, c->warp_wpc * 32, (size_t)(c->warp_smem), c->P, c->wlay, d, G, s.d_off[nxt], ox, ovx, ovy, ovz, c->d_mstate, c->d_stats, c->d_defer_count,
              c->d_defer_list, Q);
    if (auto e = check_launch(c, "shock_collide_warp", TRMCR_K_SHOCK_WARP)) return e;
  }
  prof_begin(c, TRMCR_K_SHOCK_SMEM);
  auto kern = c->smem_threads == 64 ? shock_collide_smem<Real, 64>
              : (c->smem_threads == 128 ? shock_collide_smem<Real, 128> : shock_collide_smem<Real, 256>);
  launch_k(c, kern, use_warp ? c->smem_grid : s.C, c->smem_threads, (size_t)(c->lay.total), c->P, c->lay, d, G, F, cur, fz, s.d_off[nxt], ox, ovx, ovy, ovz, c->d_mstate, c->d_stats,
      use_warp ? c->d_defer_count : nullptr, use_warp ? c->d_defer_list : nullptr, Q);
  if (auto e = check_launch(c, "shock_collide_smem", TRMCR_K_SHOCK_SMEM)) return e;
  prof_begin(c, TRMCR_K_SHOCK_GMEM);
  launch_k(c, shock_collide_gmem<Real>, c->G, c->gmem_threads, (size_t)(0), c->P, c->gs, d, G, F, cur, fz, s.d_off[nxt], ox, ovx, ovy,
                                                                 ovz, c->d_mstate, c->d_stats, Q);
  if (auto e = check_launch(c, "shock_collide_gmem", TRMCR_K_SHOCK_GMEM)) return e;
  c->cur = nxt;
  c->d_offsets = s.d_off[nxt];
  s.codes_ok = fz;     // every cell of the fused pass wrote the codes of its particles
  return TRMCR_OK;
}

// Decide (after the warp / lock-step layout is known) whether this context steps
// with the fused pass, and allocate its side data.  TRMCR_SHOCK_FUSED=1: fused
// when the lock-step kernel is available and a reservoir particle at
// |u_B| + 6 sqrt(T_B) moves less than 0.9 of a cell per step (farther movers are
// still handled, through the far-mover list, but slowly); =2 forces it; unset or
// 0: the three-pass step.  The default is the three-pass step: on C5 the fused
// pass moves 2.64 GB per step instead of 4.5 GB but takes 3.4 ms instead of
// 2.19 (its gather and move codes add ~45 % instructions to an issue-bound
// kernel, while transport and sort run at 60-75 % of DRAM bandwidth on their
// own).
inline trmcr_status shock_fused_setup(trmcr_ctx *c) {
  ShockState &s = c->shock;
  s.fused = 0;
  s.codes_ok = 0;
  const char *fe = getenv("TRMCR_SHOCK_FUSED");
  const int want = fe ? atoi(fe) : 0;
  if (want == 0 || c->lock_grid <= 0 || c->wlay.n_cap <= 0 || c->wlay.v_smem) return TRMCR_OK;
  const double vmax = std::max(fabs(s.u[0]) + 6.0 * sqrt(s.T[0]), fabs(s.u[1]) + 6.0 * sqrt(s.T[1]));
  if (want != 2 && !(vmax * c->dt * s.inv_dx <= 0.9)) return TRMCR_OK;
  s.far_cap = (int)std::min<int64_t>(std::max<int64_t>(c->cap / 64, 65536), c->cap);
  for (int k = 0; k < 2; ++k)
    if (dalloc(c, &s.d_code[k], (size_t)c->cap) || dalloc(c, &s.d_nlsr[k], sizeof(int32_t) * 3 * (size_t)s.C) ||
        dalloc(c, &s.d_far_src[k], sizeof(int32_t) * (size_t)s.far_cap) ||
        dalloc(c, &s.d_far_dst[k], sizeof(int32_t) * (size_t)s.far_cap))
      return TRMCR_ENOMEM;
  if (dalloc(c, &s.d_far_cnt, sizeof(int) * 2)) return TRMCR_ENOMEM;
  CUDA_TRY(c, cudaMemsetAsync(s.d_far_cnt, 0, sizeof(int) * 2, c->stream));
  const bool wbk = ext_variant(c);
  const void *lf = c->dtype == TRMCR_F64
                       ? (wbk ? (const void *)shock_fused_lock<double, true> : (const void *)shock_fused_lock<double, false>)
                       : (wbk ? (const void *)shock_fused_lock<float, true> : (const void *)shock_fused_lock<float, false>);
  int smem_max = 0;
  cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->dev);
  cudaFuncAttributes a;
  if (cudaFuncGetAttributes(&a, lf) != cudaSuccess ||
      cudaFuncSetAttribute(lf, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max - (int)a.sharedSizeBytes) != cudaSuccess)
    return fail(c, TRMCR_ECUDA, "cudaFuncSetAttribute(shock_fused_lock) failed");
  s.fused = 1;
  return TRMCR_OK;
}

template <typename Real>
trmcr_status shock_step(trmcr_ctx *c) {
  if (trmcr_status e = shock_begin<Real>(c)) return e;
  return shock_finish<Real>(c);
}

}  // namespace trmcr
