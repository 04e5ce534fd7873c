// device_common.cuh — counter-based RNG, keyed permutations and CTA
// reductions for the TRMC-R kernels (sm_100a).  Product code: written
// independently of oracle/ (DESIGN.md §3.1 gives the shared DEFINITIONS).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace trmcr {

// Purposes of the Philox counter word 1.
enum : uint32_t {
  kSplit = 1, kType = 2, kPerm = 3, kColl = 4, kColl2 = 5,
  kMaxw = 6, kMaxw2 = 7, kResv = 8, kResv2 = 9, kLiteral = 10
};

// Philox4x32-10: 10 rounds of the (0xD2511F53, 0xCD9E8D57) multiply-xor
// bijection with Weyl key schedule (0x9E3779B9, 0xBB67AE85).
__device__ __forceinline__ uint4 philox10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                          uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
  }
  return make_uint4(c0, c1, c2, c3);
}

// Stream identity of one cell at one step: key = seed, counter words 2,3 =
// (global cell, step); word 1 = purpose<<24 | attempt<<20 | level; word 0 = element.
// Out-of-line copy for the general kernels: one body instead of one per call
// site keeps those kernels inside the instruction cache.
__device__ __noinline__ uint4 philox10_call(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0,
                                            uint32_t k1) {
  return philox10(c0, c1, c2, c3, k0, k1);
}
struct RngKey {
  uint32_t k0, k1, cell, step;
  __device__ __forceinline__ uint4 operator()(uint32_t purpose, uint32_t attempt, uint32_t level,
                                              uint32_t elem) const {
    return philox10_call(elem, (purpose << 24) | (attempt << 20) | level, cell, step, k0, k1);
  }
};

// (k + 1/2) 2^-52 with k the top 52 bits of (hi, lo): exact, in (0,1).
__device__ __forceinline__ double u53(uint32_t hi, uint32_t lo) {
  const uint64_t k = (static_cast<uint64_t>(hi) << 20) | static_cast<uint64_t>(lo >> 12);
  return (static_cast<double>(k) + 0.5) * 0x1p-52;
}
// (k + 1/2) 2^-23 with k the top 23 bits of w: exact in fp32, in (0,1).
__device__ __forceinline__ float u24(uint32_t w) {
  return (static_cast<float>(w >> 9) + 0.5f) * 0x1p-23f;
}

// ---- keyed bijection of [0, N): Feistel on Z_A x Z_C + cycle walking ----
__device__ __forceinline__ uint32_t mix32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du;
  x ^= x >> 15; x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}

// Domain A C with A = ceil(sqrt N), C = ceil(N / A) (N <= A C < N + A, so the
// walk rarely repeats); x = L C + R.  Round i: (L, R) <- (R, (L + f_i(R)) mod
// |L|), f_i(R) = umulhi(mix32(R ^ k_i), |L|), k_i = key[i & 3] + (i >> 2)
// 0x9E3779B9; 16 rounds for N <= 64, else 8 (R17).  The state stays
// split (L, R) through the walk, so only the first split divides (by
// multiply-high with one correction step, exact for every 32-bit x).
struct PermDom {
  uint32_t N, A, C, m;   // m = floor(2^32 / C) (0 when C == 1)
};
__device__ __forceinline__ PermDom perm_dom(uint32_t n) {
  PermDom D;
  D.N = n;
  if (n <= 1u) { D.A = 1u; D.C = 1u; D.m = 0u; return D; }
  uint32_t a = (uint32_t)sqrtf((float)n);
  while ((uint64_t)a * a < n) ++a;
  while (a > 1u && (uint64_t)(a - 1u) * (a - 1u) >= n) --a;
  D.A = a;
  D.C = (n + a - 1u) / a;
  D.m = D.C == 1u ? 0u : (uint32_t)((1ull << 32) / D.C);
  return D;
}
// One round on (L in Z_wl, R): (L, R) <- (R, (L + f(R)) mod wl).  The
// reduction is min(t, t - wl) (t < 2 wl: t - wl wraps above t when t < wl).
__device__ __forceinline__ void perm_round(uint32_t &L, uint32_t &R, uint32_t k, uint32_t wl) {
  const uint32_t t = L + __umulhi(mix32(R ^ k), wl);
  L = R;
  R = min(t, t - wl);
}
__device__ __forceinline__ void perm_rounds(uint32_t &L, uint32_t &R, const uint4 &rk, const PermDom &D) {
  const int groups = D.N <= 64u ? 4 : 2;             // 16 or 8 rounds
  uint32_t kadd = 0u;
  for (int g = 0; g < groups; ++g, kadd += 0x9E3779B9u) {
    perm_round(L, R, rk.x + kadd, D.A);
    perm_round(L, R, rk.y + kadd, D.C);
    perm_round(L, R, rk.z + kadd, D.A);
    perm_round(L, R, rk.w + kadd, D.C);
  }
}
__device__ __forceinline__ void perm_split(uint32_t x, const PermDom &D, uint32_t &L, uint32_t &R) {
  if (D.C == 1u) { L = x; R = 0u; return; }
  uint32_t q = __umulhi(x, D.m);
  uint32_t r = x - q * D.C;
  if (r >= D.C) { ++q; r -= D.C; }
  L = q; R = r;
}

struct Perm {
  uint4 rk;
  PermDom D;
  __device__ __forceinline__ void init(uint4 key, uint32_t n) { rk = key; D = perm_dom(n); }
  // Cycle walking.  Out-of-range input or a walk longer than 4096 (impossible
  // for x < N) returns 0xFFFFFFFF.
  __device__ __forceinline__ uint32_t operator()(uint32_t x) const {
    if (D.N <= 1u) return x < D.N || D.N == 0u ? x : 0xFFFFFFFFu;
    if (x >= D.N) return 0xFFFFFFFFu;
    uint32_t L, R;
    perm_split(x, D, L, R);
    for (int it = 0;; ++it) {
      if (it > 4096) return 0xFFFFFFFFu;
      perm_rounds(L, R, rk, D);
      const uint32_t y = L * D.C + R;
      if (y < D.N) return y;
    }
  }
};

// Two evaluations (x_s under key k_s on domain D_s) with their cycle walks
// interleaved: the warp pays max(walk_0, walk_1) passes, not the sum, and the
// two chains are independent work for the scheduler.  Results as Perm().
__device__ __forceinline__ void perm_eval2(uint32_t x0, const uint4 &k0, const PermDom &D0, uint32_t x1,
                                           const uint4 &k1, const PermDom &D1, uint32_t &y0, uint32_t &y1) {
  const bool t0 = D0.N <= 1u || x0 >= D0.N, t1 = D1.N <= 1u || x1 >= D1.N;   // trivial / invalid
  bool w0 = !t0, w1 = !t1;
  y0 = t0 ? (x0 < D0.N ? x0 : 0xFFFFFFFFu) : 0u;
  y1 = t1 ? (x1 < D1.N ? x1 : 0xFFFFFFFFu) : 0u;
  uint32_t L0 = 0, R0 = 0, L1 = 0, R1 = 0;
  if (w0) perm_split(x0, D0, L0, R0);
  if (w1) perm_split(x1, D1, L1, R1);
  for (int it = 0; w0 || w1; ++it) {
    if (it > 4096) { if (w0) y0 = 0xFFFFFFFFu; if (w1) y1 = 0xFFFFFFFFu; break; }
    if (w0) { perm_rounds(L0, R0, k0, D0); y0 = L0 * D0.C + R0; w0 = y0 >= D0.N; }
    if (w1) { perm_rounds(L1, R1, k1, D1); y1 = L1 * D1.C + R1; w1 = y1 >= D1.N; }
  }
}

// ---- programmatic dependent launch (PDL) ----
// Every kernel of the step starts with pdl_wait(): it returns once the
// preceding kernel in the stream has completed and its writes are visible
// (a no-op when the kernel was launched without the PDL attribute), so the
// data dependencies are those of plain stream order.  pdl_trigger() lets the
// next kernel be scheduled (its launch latency overlaps this kernel).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---- CTA reductions (fixed order: reproducible run to run) ----
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
// out-of-line versions (general warp kernel: code size)
__device__ __noinline__ double warp_sum_call(double v) { return warp_sum(v); }
__device__ __noinline__ double warp_max_call(double v) { return warp_max(v); }

// Sums NV doubles over the CTA; every thread receives the totals.
// `red` must hold (blockDim.x/32)*NV doubles of shared memory.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double *red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = warp_sum(v[k]);
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) red[warp * NV + k] = v[k];
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double s = 0.0;
    for (int w = 0; w < nw; ++w) s += red[w * NV + k];
    v[k] = s;
  }
  __syncthreads();
}

__device__ __forceinline__ double block_max(double v, double *red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_max(v);
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < nw; ++w) s = fmax(s, red[w]);
  __syncthreads();
  return s;
}

}  // namespace trmcr
