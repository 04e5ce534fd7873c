// thermal.cuh — warp-per-cell fast path of the collision step for cells in
// the fluid regime, where the split (Alg 4.2) provably assigns
// every particle to N_{m+1}: p n < 2^-53 makes every IR draw exactly 0
// (DESIGN.md §3.2), so the step is "replace the cell by a Maxwellian with its
// own momentum and energy" (AP property (ii); conservative
// sampling P:558-561).  No tree, no permutation: Theta is every slot.
//
// One warp owns one cell at a time (persistent grid); the cell is staged in
// the warp's shared-memory slab, reductions are warp butterflies (bitwise
// identical on every lane), and no CTA barrier is needed.  A cell that is not
// in this regime (or larger than the slab) is queued, untouched, for the
// general kernel (cell_step.cuh).  Results equal the general path's: same
// keyed draws, same formulas.
#pragma once
#include "cell_step.cuh"

namespace trmcr {

template <typename Real> struct ThermalCap;
template <> struct ThermalCap<float> { static constexpr int value = 1024; };
template <> struct ThermalCap<double> { static constexpr int value = 512; };
#ifndef TRMCR_THERMAL_WARPS
#define TRMCR_THERMAL_WARPS 1
#endif
constexpr int kThermalWarps = TRMCR_THERMAL_WARPS;   // one warp per CTA, 16 CTAs per SM: measured 97.2 us vs 101.1 (8 warps x 2 CTAs) on C3

// 16-byte vector of Real (4 floats or 2 doubles) for coalesced, batched I/O.
template <typename Real> struct Vec;
template <> struct Vec<float> { using T = float4; static constexpr int W = 4; };
template <> struct Vec<double> { using T = double2; static constexpr int W = 2; };
template <typename V, typename Real> __device__ __forceinline__ Real vget(const V &v, int k);
template <> __device__ __forceinline__ float vget<float4, float>(const float4 &v, int k) {
  return k == 0 ? v.x : (k == 1 ? v.y : (k == 2 ? v.z : v.w));
}
template <> __device__ __forceinline__ double vget<double2, double>(const double2 &v, int k) {
  return k == 0 ? v.x : v.y;
}
template <typename V, typename Real> __device__ __forceinline__ void vset(V &v, int k, Real a);
template <> __device__ __forceinline__ void vset<float4, float>(float4 &v, int k, float a) {
  if (k == 0) v.x = a; else if (k == 1) v.y = a; else if (k == 2) v.z = a; else v.w = a;
}
template <> __device__ __forceinline__ void vset<double2, double>(double2 &v, int k, double a) {
  if (k == 0) v.x = a; else v.y = a;
}

// Moments of the staged cell (pass 2) and the thermal decision; returns true
// when the cell is in the fluid regime (p n < 2^-53).
struct ThermalMoments {
  double Sx, Sy, Sz, ux, uy, uz, E, S0, sigma, mu, p;
};

template <typename Real>
__device__ __forceinline__ void thermal_finish(const StepParams &P, const ThermalMoments &M, int n, int c,
                                               int32_t *m_state, double *stats) {
  // A7 in closed form: every retry plan is empty, E1 is fixed.
  int m = P.adaptive ? m_state[c] : P.m_fixed;
  int r = 0;
  double S_est = M.S0, E1 = 0.0;
  int m_next = m;
  if (P.adaptive) {
    const double T = M.E / (3.0 * n);
    if (P.indicator == TRMCR_IND_PXX) {
      S_est = T;
    } else {
      const double u2 = M.ux * M.ux + M.uy * M.uy + M.uz * M.uz;
      S_est = u2 * u2 + 10.0 * u2 * T + 15.0 * T * T;
    }
    E1 = M.S0 != 0.0 ? fabs(S_est - M.S0) / fabs(M.S0) : (S_est == 0.0 ? 0.0 : INFINITY);
    while (E1 > P.delta2 && m < P.m_cap) { m = 2 * m < P.m_cap ? 2 * m : P.m_cap; ++r; }
    m_next = E1 < P.delta1 ? (m / 2 > 1 ? m / 2 : 1) : m;
    m_state[c] = m_next;
  }
  double *s = stats + (size_t)c * TRMCR_NSTATS;
  s[TRMCR_ST_N] = n; s[TRMCR_ST_P] = M.p; s[TRMCR_ST_MU] = M.mu; s[TRMCR_ST_SIGMA] = M.sigma;
  s[TRMCR_ST_S0] = M.S0; s[TRMCR_ST_SEST] = S_est; s[TRMCR_ST_E1] = E1;
  s[TRMCR_ST_MUSED] = m; s[TRMCR_ST_MNEXT] = m_next; s[TRMCR_ST_DEPTH] = m;
  s[TRMCR_ST_ATTEMPTS] = r + 1; s[TRMCR_ST_LEAVES] = 0; s[TRMCR_ST_UNTOUCHED] = 0;
  s[TRMCR_ST_THERMALISED] = n; s[TRMCR_ST_PROPOSALS] = 0; s[TRMCR_ST_ACCEPTED] = 0;
  s[TRMCR_ST_VIOLATIONS] = 0; s[TRMCR_ST_MAXW] = n >= 2 ? n : 0;
  s[TRMCR_ST_PX] = M.Sx; s[TRMCR_ST_PY] = M.Sy; s[TRMCR_ST_PZ] = M.Sz;
  s[TRMCR_ST_ENERGY] = M.E + n * (M.ux * M.ux + M.uy * M.uy + M.uz * M.uz);
}

__device__ __forceinline__ void thermal_decide(const StepParams &P, ThermalMoments &M, int n, double PXX,
                                               double M4, double dv2) {
  M.S0 = (P.indicator == TRMCR_IND_PXX ? PXX : M4) / n;
  M.sigma = 0.0;
  M.mu = 1.0;
  if (P.model == TRMCR_HARD_SPHERE) { M.sigma = 2.0 * sqrt(dv2); M.mu = M.sigma; }
  else if (P.model == TRMCR_VHS) { M.sigma = vhs_majorant(dv2, P.alpha); M.mu = M.sigma; }
  M.p = exp(-(M.mu * P.dt / P.eps));
}

// Vector path: cell start and length multiples of the vector width.  Each lane
// owns whole 16-byte groups; loads/stores are 16 B per lane (512 B per warp
// instruction), the Box-Muller draws of a group are independent (ILP).
template <typename Real, int CAP>
__device__ __forceinline__ bool thermal_cell_vec(const StepParams &P, Real *vx, Real *vy, Real *vz,
                                                 int64_t off, int n, int c, Real *wx, Real *wy, Real *wz,
                                                 int32_t *m_state, double *stats) {
  using V = typename Vec<Real>::T;
  constexpr int W = Vec<Real>::W;
  constexpr int G = CAP / W / 32;          // groups per lane at n = CAP
  const int lane = threadIdx.x & 31;
  const int ng = n / W;
  V *gx = reinterpret_cast<V *>(vx + off), *gy = reinterpret_cast<V *>(vy + off), *gz = reinterpret_cast<V *>(vz + off);
  V *sx4 = reinterpret_cast<V *>(wx), *sy4 = reinterpret_cast<V *>(wy), *sz4 = reinterpret_cast<V *>(wz);
  // pass 1: batched 16-byte loads (all in flight), stage + sums
  double sx = 0, sy = 0, sz = 0;
#pragma unroll
  for (int k = 0; k < G; ++k) {
    const int g = lane + 32 * k;
    if (g < ng) {
      const V a = __ldcs(gx + g), b = __ldcs(gy + g), d = __ldcs(gz + g);
      sx4[g] = a; sy4[g] = b; sz4[g] = d;
#pragma unroll
      for (int w = 0; w < W; ++w) { sx += vget<V, Real>(a, w); sy += vget<V, Real>(b, w); sz += vget<V, Real>(d, w); }
    }
  }
  ThermalMoments M;
  M.Sx = warp_sum(sx); M.Sy = warp_sum(sy); M.Sz = warp_sum(sz);
  M.ux = M.Sx / n; M.uy = M.Sy / n; M.uz = M.Sz / n;
  const Real rux = (Real)M.ux, ruy = (Real)M.uy, ruz = (Real)M.uz;
  double e = 0, pxx = 0, m4 = 0;
  Real mx = 0;
#pragma unroll 4
  for (int g = lane; g < ng; g += 32) {
    const V a = sx4[g], b = sy4[g], d = sz4[g];
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const Real x = vget<V, Real>(a, w), y = vget<V, Real>(b, w), z = vget<V, Real>(d, w);
      const Real dx = x - rux, dy = y - ruy, dz = z - ruz;
      const Real r2 = dx * dx + dy * dy + dz * dz;
      e += r2;
      mx = r2 > mx ? r2 : mx;
      pxx += dx * dx;
      const Real v2 = x * x + y * y + z * z;
      m4 += v2 * v2;
    }
  }
  M.E = warp_sum(e);
  thermal_decide(P, M, n, warp_sum(pxx), warp_sum(m4), warp_max((double)mx));
  if (!(M.p * (double)n < 0x1p-53)) return false;
  const RngKey K{P.k0, P.k1, P.cell_base + (uint32_t)c, P.step};
  if (n >= 2) {
    double ax = 0, ay = 0, az = 0, a2 = 0;
#pragma unroll 2
    for (int g = lane; g < ng; g += 32) {
      V a, b, d;
#pragma unroll
      for (int w = 0; w < W; ++w) {
        Real g0, g1, g2;
        gauss3<Real>(K, (uint32_t)(g * W + w), g0, g1, g2);
        vset<V, Real>(a, w, g0); vset<V, Real>(b, w, g1); vset<V, Real>(d, w, g2);
        ax += g0; ay += g1; az += g2;
        a2 += (double)(g0 * g0 + g1 * g1 + g2 * g2);
      }
      sx4[g] = a; sy4[g] = b; sz4[g] = d;
    }
    const double Gx = warp_sum(ax) / n, Gy = warp_sum(ay) / n, Gz = warp_sum(az) / n;
    const double D = warp_sum(a2) - n * (Gx * Gx + Gy * Gy + Gz * Gz);
    const double sc = (D > 0.0 && M.E > 0.0) ? sqrt(M.E / D) : 0.0;
    const Real rs = (Real)sc, rgx = (Real)Gx, rgy = (Real)Gy, rgz = (Real)Gz;
#pragma unroll 4
    for (int g = lane; g < ng; g += 32) {
      V a = sx4[g], b = sy4[g], d = sz4[g];
#pragma unroll
      for (int w = 0; w < W; ++w) {
        vset<V, Real>(a, w, rux + rs * (vget<V, Real>(a, w) - rgx));
        vset<V, Real>(b, w, ruy + rs * (vget<V, Real>(b, w) - rgy));
        vset<V, Real>(d, w, ruz + rs * (vget<V, Real>(d, w) - rgz));
      }
      __stcs(gx + g, a); __stcs(gy + g, b); __stcs(gz + g, d);
    }
  }
  if (lane == 0) thermal_finish<Real>(P, M, n, c, m_state, stats);
  return true;
}

// Scalar path for unaligned cells.
template <typename Real>
__device__ __forceinline__ bool thermal_cell_scalar(const StepParams &P, Real *vx, Real *vy, Real *vz,
                                                    int64_t off, int n, int c, Real *wx, Real *wy, Real *wz,
                                                    int32_t *m_state, double *stats) {
  const int lane = threadIdx.x & 31;
  double sx = 0, sy = 0, sz = 0;
#pragma unroll 4
  for (int i = lane; i < n; i += 32) {
    const Real a = vx[off + i], b = vy[off + i], d = vz[off + i];
    wx[i] = a; wy[i] = b; wz[i] = d;
    sx += a; sy += b; sz += d;
  }
  ThermalMoments M;
  M.Sx = warp_sum(sx); M.Sy = warp_sum(sy); M.Sz = warp_sum(sz);
  M.ux = M.Sx / n; M.uy = M.Sy / n; M.uz = M.Sz / n;
  const Real rux = (Real)M.ux, ruy = (Real)M.uy, ruz = (Real)M.uz;
  double e = 0, pxx = 0, m4 = 0;
  Real mx = 0;
  for (int i = lane; i < n; i += 32) {
    const Real x = wx[i], y = wy[i], z = wz[i];
    const Real dx = x - rux, dy = y - ruy, dz = z - ruz;
    const Real r2 = dx * dx + dy * dy + dz * dz;
    e += r2;
    mx = r2 > mx ? r2 : mx;
    pxx += dx * dx;
    const Real v2 = x * x + y * y + z * z;
    m4 += v2 * v2;
  }
  M.E = warp_sum(e);
  thermal_decide(P, M, n, warp_sum(pxx), warp_sum(m4), warp_max((double)mx));
  if (!(M.p * (double)n < 0x1p-53)) return false;
  const RngKey K{P.k0, P.k1, P.cell_base + (uint32_t)c, P.step};
  if (n >= 2) {
    double gx = 0, gy = 0, gz = 0, g2 = 0;
    for (int i = lane; i < n; i += 32) {
      Real a, b, d;
      gauss3<Real>(K, (uint32_t)i, a, b, d);
      wx[i] = a; wy[i] = b; wz[i] = d;
      gx += a; gy += b; gz += d;
      g2 += (double)(a * a + b * b + d * d);
    }
    const double Gx = warp_sum(gx) / n, Gy = warp_sum(gy) / n, Gz = warp_sum(gz) / n;
    const double D = warp_sum(g2) - n * (Gx * Gx + Gy * Gy + Gz * Gz);
    const double sc = (D > 0.0 && M.E > 0.0) ? sqrt(M.E / D) : 0.0;
    const Real rs = (Real)sc, rgx = (Real)Gx, rgy = (Real)Gy, rgz = (Real)Gz;
    for (int i = lane; i < n; i += 32) {
      vx[off + i] = rux + rs * (wx[i] - rgx);
      vy[off + i] = ruy + rs * (wy[i] - rgy);
      vz[off + i] = ruz + rs * (wz[i] - rgz);
    }
  }
  if (lane == 0) thermal_finish<Real>(P, M, n, c, m_state, stats);
  return true;
}

// ---- fp32 production path (C3-class cells): cp.async staging, fp32 lane sums ----
__device__ __forceinline__ void cp_async16(void *smem_dst, const void *gmem_src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem_src) : "memory");
}
// Bulk prefetch of a contiguous global range into L2 (sm_90+): one instruction
// per array, used to pull the warp's next cell in while it works on this one.
__device__ __forceinline__ void prefetch_l2(const void *p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}
// (k + 1/2) 2^-23 for k = w >> 9, built from the mantissa bits (no I2F):
// b = 1 + k 2^-23 in [1,2); b - (1 - 2^-24) = (2k+1) 2^-24 is representable, so
// the single FADD is exact and the value is bit-identical to u24().
__device__ __forceinline__ float u24_bits(uint32_t w) {
  return __uint_as_float(0x3F800000u | (w >> 9)) + (-1.0f + 0x1p-24f);
}
// Box-Muller for the statistical fp32 path: MUFU lg2 / rsqrt / sin / cos.
// r = sqrt(-2 ln u) = a rsqrt(a), a = (-2 ln 2) log2(u) > 0 since u < 1.
__device__ __forceinline__ void gauss3_fast(const RngKey &K, uint32_t slot, float &g0, float &g1, float &g2) {
  const uint4 w = K(kMaxw, 0, 0, slot);
  const float u1 = u24_bits(w.x), u2 = u24_bits(w.y), u3 = u24_bits(w.z), u4 = u24_bits(w.w);
  constexpr float kM2Ln2 = -1.3862943611198906f;   // -2 ln 2
  const float a1 = kM2Ln2 * __log2f(u1), a3 = kM2Ln2 * __log2f(u3);
  const float r1 = a1 * rsqrtf(a1), r3 = a3 * rsqrtf(a3);
  float s2, c2;
  __sincosf(6.283185307179586f * u2, &s2, &c2);
  const float c4 = __cosf(6.283185307179586f * u4);
  g0 = r1 * c2; g1 = r1 * s2; g2 = r3 * c4;
}

__device__ __forceinline__ float2 lo2(const float4 &a) { return make_float2(a.x, a.y); }
__device__ __forceinline__ float2 hi2(const float4 &a) { return make_float2(a.z, a.w); }
__device__ __forceinline__ float4 f4(const float2 &l, const float2 &h) { return make_float4(l.x, l.y, h.x, h.y); }

// Raw MUFU approximations (flush-to-zero, no special-case fix-ups): every
// operand below is a normal number (u in [2^-24, 1), a in [1.2e-7, 23.1],
// 2 pi u in (0, 2 pi)), so the fix-up code the compiler adds around
// __log2f / rsqrtf would never fire.
__device__ __forceinline__ float lg2_ftz(float x) {
  float y; asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y;
}
__device__ __forceinline__ float rsqrt_ftz(float x) {
  float y; asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y;
}
__device__ __forceinline__ float sin_ftz(float x) {
  float y; asm("sin.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y;
}
__device__ __forceinline__ float cos_ftz(float x) {
  float y; asm("cos.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y;
}

// Box-Muller pair from two 24-bit uniforms (fp32 statistical path), scaled by
// the constant 1/sqrt(2 ln 2): r = sqrt(-log2 u) instead of sqrt(-2 ln u).
// The Maxwellian is built by shift-and-rescale to the cell's own energy
// (v' = u + s (g - G), s = sqrt(E / sum|g - G|^2)), so a common scale of all
// g cancels exactly (up to rounding) and its multiply is dropped.
// 2 pi u2 = 2 pi (b - (1 - 2^-24)) is one FFMA from the mantissa word b.
__device__ __forceinline__ void bm_pair(uint32_t wa, uint32_t wb, float &c, float &s) {
  constexpr float k2Pi = 6.283185307179586f;
  const float l = lg2_ftz(u24_bits(wa));           // log2 u < 0
  const float r = -l * rsqrt_ftz(-l);
  const float b = __uint_as_float(0x3F800000u | (wb >> 9));
  const float t = fmaf(b, k2Pi, -k2Pi * (1.0f - 0x1p-24f));
  const float2 cs = __fmul2_rn(make_float2(cos_ftz(t), sin_ftz(t)), make_float2(r, r));
  c = cs.x;
  s = cs.y;
}

// Philox4x32 with the key schedule precomputed on the host (kernel
// parameter, i.e. constant bank: the key XORs cost no extra instruction) and
// counter words 1..3 fixed per cell.  The fp32 fluid-regime draws (a
// statistical mode) use 7 rounds - Philox4x32-7 is
// Crush-resistant (Salmon et al., SC'11; 10 is Random123's safety-margin
// default) and the RNG is ~45 % of this kernel's instructions; everything else
// (fp64 parity draws, fp32 trees) keeps philox10().
#ifndef TRMCR_THERMAL_ROUNDS
#define TRMCR_THERMAL_ROUNDS 7
#endif
struct KeySched {
  uint32_t k0[10], k1[10];
};
__device__ __forceinline__ uint4 philox_ks(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                             const KeySched &ks) {
#pragma unroll
  for (int r = 0; r < TRMCR_THERMAL_ROUNDS; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    const uint32_t n0 = hi1 ^ c1 ^ ks.k0[r], n2 = hi0 ^ c3 ^ ks.k1[r];
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
  }
  return make_uint4(c0, c1, c2, c3);
}

// 12 standard normals for the 4 consecutive slots of float4 group g: three
// Philox blocks (MAXW, element 3g..3g+2) -> 6 Box-Muller pairs (fp32 mode's
// draw definition for the fluid-regime path).
__device__ __forceinline__ void gauss12(const KeySched &ks, uint32_t cell, uint32_t step, uint32_t g, float4 &a,
                                        float4 &b, float4 &d) {
  const uint32_t c1 = kMaxw << 24;
  const uint4 w0 = philox_ks(3 * g, c1, cell, step, ks), w1 = philox_ks(3 * g + 1, c1, cell, step, ks),
              w2 = philox_ks(3 * g + 2, c1, cell, step, ks);
  bm_pair(w0.x, w0.y, a.x, b.x);
  bm_pair(w0.z, w0.w, d.x, a.y);
  bm_pair(w1.x, w1.y, b.y, d.y);
  bm_pair(w1.z, w1.w, a.z, b.z);
  bm_pair(w2.x, w2.y, d.z, a.w);
  bm_pair(w2.z, w2.w, b.w, d.w);
}

// The fluid-regime step of one fp32 cell already staged (and visible to the
// whole warp) in the slab (wx, wy, wz): moments, decision, Gaussians (into
// the slab), conservative rescale, stores.  Returns false (nothing written)
// when the cell is not in the fluid regime.
__device__ __forceinline__ bool thermal_f32_compute(const StepParams &P, const KeySched &ks, float *vx, float *vy,
                                                    float *vz, int64_t off, int n, int c, float *wx, float *wy,
                                                    float *wz, int32_t *m_state, double *stats) {
  constexpr int CAP = ThermalCap<float>::value;
  constexpr int G = CAP / 4 / 32;                 // float4 groups per lane at n = CAP
  const int lane = threadIdx.x & 31;
  const int ng = n >> 2;
  float4 *gx = reinterpret_cast<float4 *>(vx + off), *gy = reinterpret_cast<float4 *>(vy + off);
  float4 *gz = reinterpret_cast<float4 *>(vz + off);
  float4 *sx4 = reinterpret_cast<float4 *>(wx), *sy4 = reinterpret_cast<float4 *>(wy);
  float4 *sz4 = reinterpret_cast<float4 *>(wz);
  // fp32 math below in packed pairs (FADD2 / FMUL2 / FFMA2: two lanes of
  // IEEE fp32 per instruction, sm_100)
  float2 s2x = make_float2(0.f, 0.f), s2y = s2x, s2z = s2x;
#pragma unroll
  for (int k = 0; k < G; ++k) {
    const int g = lane + 32 * k;
    if (g < ng) {
      const float4 a = sx4[g], b = sy4[g], d = sz4[g];
      s2x = __fadd2_rn(__fadd2_rn(s2x, lo2(a)), hi2(a));
      s2y = __fadd2_rn(__fadd2_rn(s2y, lo2(b)), hi2(b));
      s2z = __fadd2_rn(__fadd2_rn(s2z, lo2(d)), hi2(d));
    }
  }
  ThermalMoments M;
  M.Sx = warp_sum((double)(s2x.x + s2x.y)); M.Sy = warp_sum((double)(s2y.x + s2y.y));
  M.Sz = warp_sum((double)(s2z.x + s2z.y));
  M.ux = M.Sx / n; M.uy = M.Sy / n; M.uz = M.Sz / n;
  const float rux = (float)M.ux, ruy = (float)M.uy, ruz = (float)M.uz;
  const float2 nux = make_float2(-rux, -rux), nuy = make_float2(-ruy, -ruy), nuz = make_float2(-ruz, -ruz);
  float2 e2 = make_float2(0.f, 0.f), p2 = e2, q2 = e2;
  float mx = 0;
  const bool want_m4 = P.indicator == TRMCR_IND_M4;
#pragma unroll
  for (int k = 0; k < G; ++k) {
    const int g = lane + 32 * k;
    if (g < ng) {
      const float4 a = sx4[g], b = sy4[g], d = sz4[g];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const float2 xh = h ? hi2(a) : lo2(a), yh = h ? hi2(b) : lo2(b), zh = h ? hi2(d) : lo2(d);
        const float2 dx = __fadd2_rn(xh, nux), dy = __fadd2_rn(yh, nuy), dz = __fadd2_rn(zh, nuz);
        const float2 px = __fmul2_rn(dx, dx);
        const float2 r2 = __ffma2_rn(dz, dz, __ffma2_rn(dy, dy, px));
        e2 = __fadd2_rn(e2, r2);
        p2 = __fadd2_rn(p2, px);
        mx = fmaxf(mx, fmaxf(r2.x, r2.y));
        if (want_m4) {
          const float2 v2 = __ffma2_rn(zh, zh, __ffma2_rn(yh, yh, __fmul2_rn(xh, xh)));
          q2 = __ffma2_rn(v2, v2, q2);
        }
      }
    }
  }
  M.E = warp_sum((double)(e2.x + e2.y));
  thermal_decide(P, M, n, warp_sum((double)(p2.x + p2.y)), warp_sum((double)(q2.x + q2.y)), warp_max((double)mx));
  if (!(M.p * (double)n < 0x1p-53)) return false;
  const uint32_t gcell = P.cell_base + (uint32_t)c;
  if (n >= 2) {
    float2 ax = make_float2(0.f, 0.f), ay = ax, az = ax, a2 = ax;
#pragma unroll 2
    for (int k = 0; k < G; ++k) {
      const int g = lane + 32 * k;
      if (g < ng) {
        float4 a, b, d;
#ifdef TRMCR_THERMAL_NOGAUSS   // roofline experiment only: no draws
        a = make_float4(g, 1, 2, 3); b = a; d = a;
#else
        gauss12(ks, gcell, P.step, (uint32_t)g, a, b, d);
#endif
        sx4[g] = a; sy4[g] = b; sz4[g] = d;
        ax = __fadd2_rn(__fadd2_rn(ax, lo2(a)), hi2(a));
        ay = __fadd2_rn(__fadd2_rn(ay, lo2(b)), hi2(b));
        az = __fadd2_rn(__fadd2_rn(az, lo2(d)), hi2(d));
        a2 = __ffma2_rn(lo2(a), lo2(a), a2); a2 = __ffma2_rn(hi2(a), hi2(a), a2);
        a2 = __ffma2_rn(lo2(b), lo2(b), a2); a2 = __ffma2_rn(hi2(b), hi2(b), a2);
        a2 = __ffma2_rn(lo2(d), lo2(d), a2); a2 = __ffma2_rn(hi2(d), hi2(d), a2);
      }
    }
    const double Gx = warp_sum((double)(ax.x + ax.y)) / n, Gy = warp_sum((double)(ay.x + ay.y)) / n;
    const double Gz = warp_sum((double)(az.x + az.y)) / n;
    const double D = warp_sum((double)(a2.x + a2.y)) - n * (Gx * Gx + Gy * Gy + Gz * Gz);
    const double sc = (D > 0.0 && M.E > 0.0) ? sqrt(M.E / D) : 0.0;
    // v' = u + s (g - G) = s g + (u - s G): one FFMA per component
    const float rs = (float)sc;
    const float bx = (float)(M.ux - sc * Gx), by = (float)(M.uy - sc * Gy), bz = (float)(M.uz - sc * Gz);
    const float2 rs2 = make_float2(rs, rs), bx2 = make_float2(bx, bx), by2 = make_float2(by, by);
    const float2 bz2 = make_float2(bz, bz);
    __syncwarp();
#pragma unroll
    for (int k = 0; k < G; ++k) {
      const int g = lane + 32 * k;
      if (g < ng) {
        const float4 a = sx4[g], b = sy4[g], d = sz4[g];
        __stcs(gx + g, f4(__ffma2_rn(rs2, lo2(a), bx2), __ffma2_rn(rs2, hi2(a), bx2)));
        __stcs(gy + g, f4(__ffma2_rn(rs2, lo2(b), by2), __ffma2_rn(rs2, hi2(b), by2)));
        __stcs(gz + g, f4(__ffma2_rn(rs2, lo2(d), bz2), __ffma2_rn(rs2, hi2(d), bz2)));
      }
    }
  }
  if (lane == 0) thermal_finish<float>(P, M, n, c, m_state, stats);
  return true;
}

// cp.async staging of one aligned fp32 cell into the slab (one commit group).
__device__ __forceinline__ void thermal_stage_f32(const float *vx, const float *vy, const float *vz, int64_t off,
                                                  int n, float *wx, float *wy, float *wz) {
  constexpr int G = ThermalCap<float>::value / 4 / 32;
  const int lane = threadIdx.x & 31;
  const int ng = n >> 2;
  const float4 *gx = reinterpret_cast<const float4 *>(vx + off), *gy = reinterpret_cast<const float4 *>(vy + off);
  const float4 *gz = reinterpret_cast<const float4 *>(vz + off);
  float4 *sx4 = reinterpret_cast<float4 *>(wx), *sy4 = reinterpret_cast<float4 *>(wy);
  float4 *sz4 = reinterpret_cast<float4 *>(wz);
#pragma unroll
  for (int k = 0; k < G; ++k) {
    const int g = lane + 32 * k;
    if (g < ng) { cp_async16(sx4 + g, gx + g); cp_async16(sy4 + g, gy + g); cp_async16(sz4 + g, gz + g); }
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}

// Stage (all 16-byte loads in flight at once), wait, L2-prefetch the warp's
// next cell, compute.
__device__ __forceinline__ bool thermal_cell_f32(const StepParams &P, const KeySched &ks, float *vx, float *vy,
                                                 float *vz, int64_t off, int n, int c, float *wx, float *wy,
                                                 float *wz, int32_t *m_state, double *stats, int64_t next_off,
                                                 int next_n) {
  const int lane = threadIdx.x & 31;
  thermal_stage_f32(vx, vy, vz, off, n, wx, wy, wz);
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncwarp();
  if (next_n > 0 && lane < 3 && ((next_off | next_n) & 3) == 0) {
    const float *base = lane == 0 ? vx : (lane == 1 ? vy : vz);
    prefetch_l2(base + next_off, (unsigned)next_n * 4u);
  }
  return thermal_f32_compute(P, ks, vx, vy, vz, off, n, c, wx, wy, wz, m_state, stats);
}

#ifndef TRMCR_THERMAL_MINB
#define TRMCR_THERMAL_MINB 16   // one-warp CTAs per SM (12 KB of staging each); 17 measured slower (C3 97.9 -> 105.6 us: 96-register cap)
#endif
template <typename Real>
__global__ void __launch_bounds__(kThermalWarps * 32, TRMCR_THERMAL_MINB)
thermal_warp_kernel(StepParams P, KeySched ks, const int64_t *__restrict__ offsets, int ncells, Real *vx,
                    Real *vy, Real *vz, int32_t *m_state, double *stats, int *defer_count, int *defer_list,
                    int prefetch, int *zero_next) {
  step_kernel_prologue(zero_next);
  constexpr int CAP = ThermalCap<Real>::value;
  constexpr int W = Vec<Real>::W;
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  Real *wx = reinterpret_cast<Real *>(smem) + (size_t)warp * 3 * CAP;
  Real *wy = wx + CAP, *wz = wy + CAP;
  const int nwarps = gridDim.x * kThermalWarps;
  int c = blockIdx.x * kThermalWarps + warp;
  int64_t off = c < ncells ? offsets[c] : 0, end = c < ncells ? offsets[c + 1] : 0;
  const bool base_al = ((reinterpret_cast<uintptr_t>(vx) | reinterpret_cast<uintptr_t>(vy) |
                         reinterpret_cast<uintptr_t>(vz)) & 15) == 0;
  for (; c < ncells; c += nwarps) {
    const int n = (int)(end - off);
    const int64_t cur_off = off;
    // prefetch the next cell's offsets of this warp (hides one global round trip)
    const int cn = c + nwarps;
    if (cn < ncells) {
      off = offsets[cn];
      end = offsets[cn + 1];
    }
    bool done = false;
    if (n > 0 && n <= CAP) {
      const bool aligned = (cur_off % W) == 0 && (n % W) == 0 && base_al;
      if constexpr (sizeof(Real) == 4) {
        const int nn = (prefetch && cn < ncells) ? (int)(end - off) : 0;
        done = aligned ? thermal_cell_f32(P, ks, vx, vy, vz, cur_off, n, c, wx, wy, wz, m_state, stats, off, nn)
                       : thermal_cell_scalar<Real>(P, vx, vy, vz, cur_off, n, c, wx, wy, wz, m_state, stats);
      } else {
        done = aligned ? thermal_cell_vec<Real, CAP>(P, vx, vy, vz, cur_off, n, c, wx, wy, wz, m_state, stats)
                       : thermal_cell_scalar<Real>(P, vx, vy, vz, cur_off, n, c, wx, wy, wz, m_state, stats);
      }
    }
    if (!done && lane == 0) defer_list[atomicAdd(defer_count, 1)] = c;   // general path
    __syncwarp();
  }
  step_kernel_epilogue();
}

}  // namespace trmcr
