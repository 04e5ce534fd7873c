// literal.cuh — the paper's own layout of the collision step, for measuring
// the level-synchronous (LS) reformulation against it.
//
// Alg 4.3/4.4 exactly as printed, one thread per cell:
// for n = m'..1, while N_n > 0, take a sample of f_n by the recursive build
// "choose k uniform in {0..n-1}; take v_i from f_k and v_j from f_{n-k-1}"
// (P:487-496): a sample of f_0 is the next particle in the keyed order pi_0; a
// stored sample of f_k is reused (the c_k counter, is 0 or 1: a sibling
// is stored only by a fresh build and consumed by the next demand); else both
// outputs of a fresh build of f_k are made, one returned, one stored
// ("N_k = N_k - 1" per stored / "+ 1" per reused sample).  Each collision is
// the A6 pair collision with the acceptance-rejection of P:546-549.  Every
// uniform comes from one sequential keyed stream (LITERAL, element = draw
// counter, two 53-bit uniforms per Philox call, second one first; DESIGN.md
// R2/R34), so an fp64 run is a fixed realisation that the tests compare
// result for result.  Then Theta = pi_0 positions
// [L, L + |Theta|) (ascending slot order) goes through the conservative
// Maxwellian (A8), as in the LS path.
//
// Recursion is an explicit per-thread stack (depth <= m' + 1 <= kLitMaxLevel).
// Fixed truncation only (no RAD / TRMC-WB), homogeneous cells.
#pragma once
#include "cell_step.cuh"

namespace trmcr {

constexpr int kLitMaxLevel = 128;
constexpr int kLitThreads = 128;
enum : int { kErrLiteralLeaves = 64 };

struct LitFrame {
  int lev, k, i, j, phase;
};

// The sequential uniform stream of the cell (LITERAL purpose).
struct LitStream {
  RngKey K;
  uint32_t ctr;
  double buf[2];
  int nbuf;
  __device__ __forceinline__ double operator()() {
    if (nbuf == 0) {
      const uint4 w = K(kLiteral, 0, 0, ctr++);
      buf[0] = u53(w.x, w.y);
      buf[1] = u53(w.z, w.w);
      nbuf = 2;
    }
    return buf[--nbuf];
  }
};

// IR at split level d with its keyed uniform (SPLIT, 0, d, 0); 0 when y < 2^-53.
__device__ __forceinline__ int64_t lit_ir(const RngKey &K, int d, double y) {
  if (y < 0x1p-53) return 0;
  const uint4 w = K(kSplit, 0, (uint32_t)d, 0);
  const double u = u53(w.x, w.y), fl = floor(y);
  return (int64_t)fl + ((u < y - fl) ? 1 : 0);
}

template <typename Real>
__global__ void __launch_bounds__(kLitThreads)
literal_step_kernel(StepParams P, const int64_t *__restrict__ offsets, int ncells, Real *vx_all, Real *vy_all,
                    Real *vz_all, double *stats, uint8_t *flag_all, double *g_all) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncells) return;
  const int64_t o0 = offsets[c], n64 = offsets[c + 1] - o0;
  const int n = (int)n64;
  Real *vx = vx_all + o0, *vy = vy_all + o0, *vz = vz_all + o0;
  uint8_t *flag = flag_all + o0;
  double *g = g_all + 3 * o0;
  double *s = stats + (size_t)c * TRMCR_NSTATS;
  const int m = P.m_fixed;
  for (int k = 0; k < TRMCR_NSTATS; ++k) s[k] = 0.0;
  s[TRMCR_ST_MUSED] = m;
  s[TRMCR_ST_MNEXT] = m;
  if (n == 0) return;
  const uint32_t gcell = (uint32_t)(P.cell_base + c);
  const RngKey K{P.k0, P.k1, gcell, P.step};

  // ---- A3: moments and majorant, sequential in slot order ----
  double sx = 0, sy = 0, sz = 0;
  for (int i = 0; i < n; ++i) { sx += (double)vx[i]; sy += (double)vy[i]; sz += (double)vz[i]; }
  const double ux = sx / n, uy = sy / n, uz = sz / n;
  double dv2 = 0, pxx = 0, m4 = 0, c2 = 0;
  for (int i = 0; i < n; ++i) {
    const double x = vx[i], y = vy[i], z = vz[i];
    const double dx = x - ux, dy = y - uy, dz = z - uz;
    const double r2 = sq3(dx, dy, dz);
    if (r2 > dv2) dv2 = r2;
    pxx += dx * dx;
    const double v2 = x * x + y * y + z * z;
    m4 += v2 * v2;
    c2 += r2;
  }
  const double S0 = (P.indicator == TRMCR_IND_PXX) ? pxx / n : m4 / n;
  double sigma = 0.0, mu = 1.0;               // rho_c = 1 (homogeneous)
  if (P.model == TRMCR_HARD_SPHERE) { sigma = 2.0 * sqrt(dv2); mu = sigma; }
  else if (P.model == TRMCR_VHS) { sigma = vhs_majorant(dv2, P.alpha); mu = sigma; }
  const double p = exp(-(mu * P.dt / P.eps));

  // ---- A4: Wild split (Alg 4.2), levels 0..m ----
  int64_t Nk[kLitMaxLevel + 1];
  int32_t store[kLitMaxLevel + 1];
  uint8_t has[kLitMaxLevel + 1];
  int64_t rem;
  {
    const double y0 = p * (double)n;
    Nk[0] = lit_ir(K, 0, y0);
    rem = n - Nk[0];
  }
  int top = 0;
  while (rem > 0 && top < m) {
    const double y = p * (double)rem;
    if (y < 0x1p-53) {
      while (top < m) Nk[++top] = 0;
      break;
    }
    ++top;
    int64_t q = lit_ir(K, top, y);
    if (q > rem) q = rem;
    Nk[top] = q;
    rem -= q;
  }
  for (int d = 0; d <= top; ++d) has[d] = 0;

  // ---- A5/A6: the recursive trees, literally ----
  Perm pi0;
  pi0.init(K(kPerm, 0, 0, 0), (uint32_t)n);
  LitStream U{K, 0u, {0.0, 0.0}, 0};
  LitFrame st[kLitMaxLevel + 2];
  int leaf = 0, err = 0;
  unsigned long long prop = 0, acc = 0;
  unsigned viol = 0;
  Real sig = (Real)sigma;
  // get(k) without a build: a particle of f_0, or the stored sample of f_k
  auto get_now = [&](int k, int &x) -> bool {
    if (k == 0) {
      if (leaf >= n) { err = 1; x = 0; return true; }
      x = (int)pi0((uint32_t)leaf++);
      return true;
    }
    if (has[k]) {
      (void)U();                               // "random choice" among c_k = 1 stored samples
      has[k] = 0;
      Nk[k] += 1;
      x = store[k];
      return true;
    }
    return false;
  };
  for (int lev = top; lev >= 1 && !err; --lev) {
    while (Nk[lev] > 0 && !err) {
      int sp = 0, ra = 0, rb = 0;
      st[sp++] = LitFrame{lev, 0, 0, 0, 0};
      while (sp > 0 && !err) {
        LitFrame &F = st[sp - 1];
        if (F.phase == 0) {                    // k uniform in {0..lev-1}; v_i from f_k
          F.k = (int)(U() * (double)F.lev);
          int x;
          if (get_now(F.k, x)) { F.i = x; F.phase = 2; }
          else { F.phase = 1; st[sp++] = LitFrame{F.k, 0, 0, 0, 0}; }
        } else if (F.phase == 1) {             // fresh build of f_k returned (ra, rb)
          store[F.k] = rb; has[F.k] = 1; Nk[F.k] -= 1;
          F.i = ra; F.phase = 2;
        } else if (F.phase == 2) {             // v_j from f_{lev-k-1}
          const int k2 = F.lev - F.k - 1;
          int x;
          if (get_now(k2, x)) { F.j = x; F.phase = 4; }
          else { F.phase = 3; st[sp++] = LitFrame{k2, 0, 0, 0, 0}; }
        } else if (F.phase == 3) {
          const int k2 = F.lev - F.k - 1;
          store[k2] = rb; has[k2] = 1; Nk[k2] -= 1;
          F.j = ra; F.phase = 4;
        } else {                               // the collision of the two samples
          const double xa = U(), xi1 = U(), xi2 = U();
          ++prop;
          Real sj = Real(0);
          if (P.sigma_update) {                // [R33]: this pair's sigma, before it collides
            const Real q = qnorm(vx[F.i] - vx[F.j], vy[F.i] - vy[F.j], vz[F.i] - vz[F.j]);
            sj = P.model == TRMCR_VHS ? RealOps<Real>::pow_(q, (Real)P.alpha) : q;
          }
          acc += pair_collide<Real>(P, vx, vy, vz, sig, (Real)xa, (Real)xi1, (Real)xi2, (uint32_t)F.i,
                                    (uint32_t)F.j, viol);
          if (P.sigma_update && sj > viol_bound(sig)) sig = sj;
          ra = F.i; rb = F.j;
          --sp;
        }
      }
      Nk[lev] -= 2;
    }
  }
  if (err) { atomicOr(P.err, kErrLiteralLeaves); return; }

  // ---- A8: Theta = pi_0 positions [L, L + |Theta|), ascending slot order ----
  const int L = leaf;
  const int U0 = Nk[0] < n - L ? (int)Nk[0] : n - L;
  const int nT = n - L - U0;
  if (nT >= 2) {
    for (int i = 0; i < n; ++i) flag[i] = 0;
    for (int q = 0; q < nT; ++q) flag[pi0((uint32_t)(L + q))] = 1;
    double px = 0, py = 0, pz = 0;
    for (int i = 0; i < n; ++i)
      if (flag[i]) { px += (double)vx[i]; py += (double)vy[i]; pz += (double)vz[i]; }
    const double mx = px / nT, my = py / nT, mz = pz / nT;
    double ec = 0, gx = 0, gy = 0, gz = 0;
    for (int i = 0; i < n; ++i)
      if (flag[i]) {
        ec += sq3((double)vx[i] - mx, (double)vy[i] - my, (double)vz[i] - mz);
        Real g0, g1, g2;
        gauss3<Real>(K, (uint32_t)i, g0, g1, g2);
        g[3 * i] = g0; g[3 * i + 1] = g1; g[3 * i + 2] = g2;
        gx += g0; gy += g1; gz += g2;
      }
    gx /= nT; gy /= nT; gz /= nT;
    double D = 0;
    for (int i = 0; i < n; ++i)
      if (flag[i]) D += sq3(g[3 * i] - gx, g[3 * i + 1] - gy, g[3 * i + 2] - gz);
    const double sc = (D > 0 && ec > 0) ? sqrt(ec / D) : 0.0;
    for (int i = 0; i < n; ++i)
      if (flag[i]) {
        vx[i] = (Real)(mx + sc * (g[3 * i] - gx));
        vy[i] = (Real)(my + sc * (g[3 * i + 1] - gy));
        vz[i] = (Real)(mz + sc * (g[3 * i + 2] - gz));
      }
  }
  s[TRMCR_ST_N] = n; s[TRMCR_ST_P] = p; s[TRMCR_ST_MU] = mu; s[TRMCR_ST_SIGMA] = sigma; s[TRMCR_ST_S0] = S0;
  s[TRMCR_ST_DEPTH] = top; s[TRMCR_ST_ATTEMPTS] = 1;
  s[TRMCR_ST_LEAVES] = L; s[TRMCR_ST_UNTOUCHED] = U0; s[TRMCR_ST_THERMALISED] = nT;
  s[TRMCR_ST_PROPOSALS] = (double)prop; s[TRMCR_ST_ACCEPTED] = (double)acc; s[TRMCR_ST_VIOLATIONS] = viol;
  s[TRMCR_ST_MAXW] = nT >= 2 ? nT : 0;
  s[TRMCR_ST_PX] = sx; s[TRMCR_ST_PY] = sy; s[TRMCR_ST_PZ] = sz;
  s[TRMCR_ST_ENERGY] = c2 + n * (ux * ux + uy * uy + uz * uz);
}

}  // namespace trmcr
