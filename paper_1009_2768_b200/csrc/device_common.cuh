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
  kMaxw = 6, kMaxw2 = 7, kResv = 8, kResv2 = 9
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
struct RngKey {
  uint32_t k0, k1, cell, step;
  __device__ __forceinline__ uint4 operator()(uint32_t purpose, uint32_t attempt, uint32_t level,
                                              uint32_t elem) const {
    return philox10(elem, (purpose << 24) | (attempt << 20) | level, cell, step, k0, k1);
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

// ---- keyed bijection of [0, N): 4-round balanced Feistel + cycle walking ----
__device__ __forceinline__ uint32_t mix32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du;
  x ^= x >> 15; x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}

// Domain 2^b, b = ceil(log2 N) (< 2N, so cycle walking takes < 2 rounds on
// average); L = high a = floor(b/2) bits, R = low c = b - a bits; round i:
// (L, R) <- (R, L ^ (mix32(R ^ k_i) mod 2^width(L))): widths alternate and are
// back to (a, c) after 4 rounds.
struct Perm {
  uint4 rk;
  uint32_t N, c, mask_a, mask_c;
  __device__ __forceinline__ void init(uint4 key, uint32_t n) {
    rk = key;
    N = n;
    const uint32_t b = n > 1 ? 32u - __clz(n - 1u) : 1u;
    const uint32_t a = b >> 1;
    c = b - a;
    mask_a = (1u << a) - 1u;
    mask_c = (c >= 32u) ? 0xFFFFFFFFu : ((1u << c) - 1u);
  }
  __device__ __forceinline__ uint32_t round4(uint32_t y) const {
    uint32_t L = y >> c, R = y & mask_c, t;
    t = L ^ (mix32(R ^ rk.x) & mask_a); L = R; R = t;   // widths (a,c) -> (c,a)
    t = L ^ (mix32(R ^ rk.y) & mask_c); L = R; R = t;   // (c,a) -> (a,c)
    t = L ^ (mix32(R ^ rk.z) & mask_a); L = R; R = t;
    t = L ^ (mix32(R ^ rk.w) & mask_c); L = R; R = t;
    return (L << c) | R;
  }
  // Cycle walking.  Out-of-range input or a walk longer than 4096 (impossible
  // for x < N) returns 0xFFFFFFFF.
  __device__ __forceinline__ uint32_t operator()(uint32_t x) const {
    if (N <= 1u) return x < N || N == 0u ? x : 0xFFFFFFFFu;
    if (x >= N) return 0xFFFFFFFFu;
    uint32_t y = round4(x);
    for (int it = 0; y >= N; ++it) {
      if (it > 4096) return 0xFFFFFFFFu;
      y = round4(y);
    }
    return y;
  }
};

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
