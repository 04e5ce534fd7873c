/*
 * trmcr_oracle.c — CPU ORACLE FOR THE TRMC-R HOT PATH.  TEST INFRASTRUCTURE ONLY.
 *
 * What it is: a plain, slow, single-threaded fp64 implementation of one
 * time step of the recursive Time-Relaxed Monte Carlo method (TRMC-R) of
 * Pareschi & Russo / Di Stefano et al., arXiv:1009.2768 ("PAPER" below; a
 * reference "P:nnn" is PAPER.md line nnn), written straight from the paper's
 * algorithms in their order and notation.  Readings of ambiguous or garbled
 * passages are listed in DESIGN.md §2 (R1..R30) and cited here as [Rnn].
 *
 * Who may use it: ONLY tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs.  The product path
 * (paper_1009_2768_b200/) never loads, links or calls this file; the two
 * share no code, headers, tables or constants generators.
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fPIC -shared (see oracle.py).
 *
 * Parity status of each function (pins live in tests/test_oracle_*.py):
 *   orc_philox4x32_10   pinned: Random123 known-answer vectors + cuRAND's
 *                       curand_Philox4x32_10 compiled for the host.
 *   orc_ir              pinned: exact two-point law, E[IR(x)] = x.
 *   orc_split           pinned: E[N_k] = (1-tau) tau^k n, E[rem] = tau^{m+1} n
 *                       (Alg 4.2 + eq. WST), exact pmf by enumeration for n<=4.
 *   orc_feistel         pinned: bijection on [0,N) (exhaustive), uniformity.
 *   orc_collide_pair    pinned: worked example (1,0,0),(-1,0,0) (eq. n3d),
 *                       invariants, isotropy E[sigma]=0, E[sigma sigma^T]=I/3.
 *   orc_maxwellian      pinned: exact prescribed moments, Gaussian law (KS).
 *   orc_step_cells      pinned: Maxwell-molecule closed forms (Pxx, M4 decay),
 *                       truncated-map R_m(tau) for m = 1..16 (pins the
 *                       plan's type law and matching independence), McKean
 *                       tree-shape law prod 1/k_v (chi^2 on levels 3-5),
 *                       C_d = ceil((N_d + cons_d)/2), conservation,
 *                       tau->0 identity, tau->1 Maxwellian (AP),
 *                       equilibrium invariance, literal Alg 4.3/4.4 = LS at
 *                       m <= 2 and != eq. WST at m >= 4 (DESIGN R2),
 *                       Sigma >= pairwise max.
 *     rad_estimate      pinned: E1 against the N -> inf closed forms (Pxx:
 *                       (1 - R_m) A_xx/(T + A_xx); M4: y_k recursion) and
 *                       S_est = E[post-step indicator] on drifting cells.
 *   orc_shock_step      pinned: reservoir inflow vs one-sided flux closed
 *                       form, stable sort vs brute force, RH plateaus;
 *                       interior shock profile: PARITY UNPINNED (no closed
 *                       form; the paper's figures are absent).
 *   orc_rankine_hugoniot pinned: textbook normal-shock values at M=3, M=5.
 */
#include "trmcr_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

/* ===================================================================== */
/* Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11), from its definition */
/* ===================================================================== */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int round = 0; round < 10; round++) {
    uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* u = (k + 1/2) 2^-52, k the 52 bits (hi << 20 | lo >> 12): exact, in (0,1). */
double orc_u53(uint32_t hi, uint32_t lo) {
  uint64_t k = ((uint64_t)hi << 20) | (uint64_t)(lo >> 12);
  return ((double)k + 0.5) * 0x1p-52;
}

typedef struct { uint64_t seed; uint32_t gcell, step; } keyctx;

/* counter = (element, purpose<<24 | attempt<<20 | level, cell, step), key = seed. */
static void draw(const keyctx *K, int purpose, int attempt, int level, uint32_t elem,
                 uint32_t out[4]) {
  uint32_t ctr[4] = {elem,
                     ((uint32_t)purpose << 24) | ((uint32_t)attempt << 20) | (uint32_t)level,
                     K->gcell, K->step};
  uint32_t key[2] = {(uint32_t)K->seed, (uint32_t)(K->seed >> 32)};
  orc_philox4x32_10(ctr, key, out);
}

/* ===================================================================== */
/* IR: stochastic integer rounding                             */
/* IR(y) = [y] w.p. [y]+1-y, [y]+1 w.p. y-[y]; realised as [y] + (u < y-[y]) */
/* ===================================================================== */
int64_t orc_ir(double y, double u) {
  double fl = floor(y);
  return (int64_t)fl + ((u < y - fl) ? 1 : 0);
}

/* IR at split level d with its own keyed uniform [R12].  When y < 2^-53 no
 * uniform u >= 2^-53 can be below y, so the result is 0 without a draw. */
static int64_t ir_split(const keyctx *K, int d, double y) {
  if (y < 0x1p-53) return 0;
  uint32_t w[4];
  draw(K, ORC_P_SPLIT, 0, d, 0, w);
  return orc_ir(y, orc_u53(w[0], w[1]));
}

/* ===================================================================== */
/* Alg 4.2: splitting into collision sets.                      */
/* With lambda_n = tau^n exactly, omega_n/lambda_n = 1 - tau = p [R11], so */
/* N_n = IR(p * Ntilde_n), Ntilde_n = remaining particles; the loop runs   */
/* WHILE Ntilde > 0 and n < m [R10]; N_{m+1} = remainder.                  */
/* ===================================================================== */
typedef struct { double p; int64_t rem; int32_t d; } split_t;

static void split_begin(const keyctx *K, split_t *s, double p, int64_t n, int64_t *N) {
  s->p = p;
  N[0] = ir_split(K, 0, p * (double)n);            /* N_0 = IR(omega_0 N / lambda_0) */
  s->rem = n - N[0];
  s->d = 0;
}

static void split_extend(const keyctx *K, split_t *s, int32_t m, int64_t *N) {
  while (s->rem > 0 && s->d < m) {
    double y = s->p * (double)s->rem;
    if (y < 0x1p-53) {                             /* every further IR is 0 */
      while (s->d < m) N[++s->d] = 0;
      break;
    }
    s->d++;
    int64_t q = ir_split(K, s->d, y);
    if (q > s->rem) q = s->rem;                    /* cannot happen for p <= 1 */
    N[s->d] = q;
    s->rem -= q;
  }
}

int32_t orc_split(double p, int64_t n, int32_t m, uint64_t seed, uint32_t gcell, uint32_t step,
                  int64_t *N_out, int64_t *rem_out) {
  keyctx K = {seed, gcell, step};
  split_t s;
  for (int i = 0; i <= m + 1; i++) N_out[i] = 0;
  split_begin(&K, &s, p, n, N_out);
  split_extend(&K, &s, m, N_out);
  N_out[m + 1] = s.rem;
  *rem_out = s.rem;
  return s.d;
}

/* ===================================================================== */
/* Keyed permutation: Feistel on a mixed-radix domain with cycle walking.  */
/* walking.  Realises "a random choice" of f_0 particles and of stored     */
/* particles as uniform draws without replacement [R17].      */
/* ===================================================================== */
static uint32_t mix32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du;
  x ^= x >> 15; x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}

/* Domain Z_A x Z_C with A = ceil(sqrt(N)), C = ceil(N / A), so that
 * N <= A C < N + A (cycle walking rejects less than 1/sqrt(N) of the points).
 * x = L C + R with L in Z_A, R in Z_C.  Round i (i = 0..R-1):
 *   (L, R) <- (R, (L + f_i(R)) mod |L|),  f_i(R) = floor(mix32(R ^ k_i) |L| / 2^32),
 * |L| the size of the half being replaced (sizes alternate; R is even, so they
 * are back to (A, C) at the end), k_i = key[i mod 4] + floor(i / 4) 0x9E3779B9
 * (mod 2^32), y = L C + R; the walk repeats the rounds until y < N.  Each
 * round is a bijection Z_A x Z_C -> Z_C x Z_A.  Rounds: R = 16 for N <= 64,
 * else 8 — fewer rounds leave a measurable pair bias (adjacent images over-
 * represented; R17, tests/test_oracle_primitives.py). */
int64_t orc_feistel(uint64_t x, uint64_t N, const uint32_t rk[4]) {
  if (N <= 1) return (int64_t)x;
  uint64_t A = 1;
  while (A * A < N) A++;
  const uint64_t C = (N + A - 1) / A;
  const int rounds = N <= 64 ? 16 : 8;
  uint64_t L = x / C, R = x % C, y;
  do {
    uint64_t wl = A, wr = C;
    for (int i = 0; i < rounds; i++) {
      const uint32_t k = rk[i & 3] + (uint32_t)(i >> 2) * 0x9E3779B9u;
      const uint64_t f = ((uint64_t)mix32((uint32_t)R ^ k) * wl) >> 32;
      uint64_t t = L + f;
      if (t >= wl) t -= wl;
      L = R;
      R = t;
      const uint64_t w = wl; wl = wr; wr = w;
    }
    y = L * C + R;
  } while (y >= N);
  return (int64_t)y;
}

/* ===================================================================== */
/* Binary collision, eq. (Maxwell_coll) P:381-385 and eq. (n3d)  */
/* cos(theta) = 2 xi1 - 1, sin(theta) = sqrt((1-c)(1+c)) [R3], phi = 2 pi xi2 */
/* ===================================================================== */
void orc_collide_pair(double *vi, double *vj, double xi1, double xi2) {
  double qx = vi[0] - vj[0], qy = vi[1] - vj[1], qz = vi[2] - vj[2];
  double q = sqrt(qx * qx + qy * qy + qz * qz);
  double c = 2.0 * xi1 - 1.0;
  double s = sqrt((1.0 - c) * (1.0 + c));
  double phi = 2.0 * M_PI * xi2;
  double sx = s * cos(phi), sy = s * sin(phi), sz = c;
  double h = 0.5 * q;
  double gx = 0.5 * (vi[0] + vj[0]), gy = 0.5 * (vi[1] + vj[1]), gz = 0.5 * (vi[2] + vj[2]);
  vi[0] = gx + h * sx; vi[1] = gy + h * sy; vi[2] = gz + h * sz;
  vj[0] = gx - h * sx; vj[1] = gy - h * sy; vj[2] = gz - h * sz;
}

/* ===================================================================== */
/* Conservative Maxwellian sampling, P:558-561 [R18]: Gaussians by         */
/* Box-Muller, then shift-and-rescale to the set's own pre-step momentum   */
/* and energy.  k == 1 keeps the particle (two moments cannot be matched). */
/* ===================================================================== */
static void gauss3(const keyctx *K, uint32_t slot, double g[3]) {
  uint32_t w[4], w2[4];
  draw(K, ORC_P_MAXW, 0, 0, slot, w);
  draw(K, ORC_P_MAXW2, 0, 0, slot, w2);
  double u1 = orc_u53(w[0], w[1]), u2 = orc_u53(w[2], w[3]);
  double u3 = orc_u53(w2[0], w2[1]), u4 = orc_u53(w2[2], w2[3]);
  double r1 = sqrt(-2.0 * log(u1)), r3 = sqrt(-2.0 * log(u3));
  g[0] = r1 * cos(2.0 * M_PI * u2);
  g[1] = r1 * sin(2.0 * M_PI * u2);
  g[2] = r3 * cos(2.0 * M_PI * u4);
}

void orc_maxwellian(int64_t k, const int64_t *slots, double *vx, double *vy, double *vz,
                    uint64_t seed, uint32_t gcell, uint32_t step) {
  if (k < 2) return;
  keyctx K = {seed, gcell, step};
  double px = 0, py = 0, pz = 0;
  for (int64_t i = 0; i < k; i++) { px += vx[slots[i]]; py += vy[slots[i]]; pz += vz[slots[i]]; }
  double ux = px / (double)k, uy = py / (double)k, uz = pz / (double)k;
  double ec = 0;
  for (int64_t i = 0; i < k; i++) {
    double dx = vx[slots[i]] - ux, dy = vy[slots[i]] - uy, dz = vz[slots[i]] - uz;
    ec += dx * dx + dy * dy + dz * dz;
  }
  double *g = (double *)malloc(sizeof(double) * 3 * (size_t)k);
  double gx = 0, gy = 0, gz = 0;
  for (int64_t i = 0; i < k; i++) {
    gauss3(&K, (uint32_t)slots[i], g + 3 * i);
    gx += g[3 * i]; gy += g[3 * i + 1]; gz += g[3 * i + 2];
  }
  gx /= (double)k; gy /= (double)k; gz /= (double)k;
  double D = 0;
  for (int64_t i = 0; i < k; i++) {
    double a = g[3 * i] - gx, b = g[3 * i + 1] - gy, c = g[3 * i + 2] - gz;
    D += a * a + b * b + c * c;
  }
  double sc = (D > 0 && ec > 0) ? sqrt(ec / D) : 0.0;
  for (int64_t i = 0; i < k; i++) {
    vx[slots[i]] = ux + sc * (g[3 * i] - gx);
    vy[slots[i]] = uy + sc * (g[3 * i + 1] - gy);
    vz[slots[i]] = uz + sc * (g[3 * i + 2] - gz);
  }
  free(g);
}

/* ===================================================================== */
/* Collision log                                                          */
/* ===================================================================== */
typedef struct { orc_coll_rec *buf; int64_t cap; int64_t n; } logger;

static void log_coll(logger *lg, uint32_t cell, int r, int d, int64_t j, int64_t si, int64_t sk,
                     int acc) {
  if (!lg) return;
  if (lg->n < lg->cap) {
    orc_coll_rec *e = &lg->buf[lg->n];
    e->cell = (int32_t)cell; e->attempt = r; e->level = d; e->accepted = acc;
    e->j = j; e->slot_i = si; e->slot_k = sk;
  }
  lg->n++;
}

/* One (possibly dummy) collision of a tree node: Alg 4.4 step 5.
 * HS: accept iff xi * Sigma' < |q| (K cancels) [R7]; a rejected pair is a
 * tree node whose particles pass through unchanged [R19]. */
typedef struct {
  const orc_params *P; keyctx K; double sigma;
  double *vx, *vy, *vz; orc_cell_stats *st; logger *lg;
} cellctx;

/* Acceptance-rejection of a dummy collision (sec. VHS): accept iff
 * xi Sigma < sigma_ij with sigma_ij = K|q|^alpha and Sigma = K (2 dv)^alpha
 * (K cancels [R7]); Sigma here is Sigma' = (2 dv)^alpha.  HS (alpha = 1)
 * compares |q| itself; Maxwell (alpha = 0) always accepts.  A violation is
 * a pair above the bound (|q|^alpha > Sigma').
 * Majorant variant (remark after Alg 4.4: "update the upper
 * bound itself, after each collision"): with sigma_update the bound becomes
 * max(Sigma, sigma_ij) after every proposal, in the canonical order (level
 * ascending, collision index ascending; RAD attempts in order) [R33]. */
static int vhs_accept(const orc_params *P, double *sigma, double q, double xa, double *viol) {
  double s;
  if (P->model == ORC_HARD_SPHERE) s = q;
  else if (P->model == ORC_VHS) s = pow(q, P->alpha);
  else return 1;
  /* a violation exceeds the bound by more than its rounding [R35]: in a
   * two-particle cell |q| = 2 max|v - u| exactly */
  const int over = s > *sigma * (1.0 + 0x1p-40);
  if (over) *viol += 1;
  const int acc = xa * *sigma < s;
  if (P->sigma_update && over) *sigma = s;
  return acc;
}

static void tree_collision(cellctx *X, int r, int d, int64_t j, int64_t si, int64_t sk) {
  uint32_t w[4], w2[4];
  draw(&X->K, ORC_P_COLL, r, d, (uint32_t)j, w);
  draw(&X->K, ORC_P_COLL2, r, d, (uint32_t)j, w2);
  double xa = orc_u53(w[0], w[1]), xi1 = orc_u53(w[2], w[3]), xi2 = orc_u53(w2[0], w2[1]);
  double vi[3] = {X->vx[si], X->vy[si], X->vz[si]};
  double vk[3] = {X->vx[sk], X->vy[sk], X->vz[sk]};
  int acc = 1;
  X->st->proposals += 1;
  if (X->P->model != ORC_MAXWELL) {
    double qx = vi[0] - vk[0], qy = vi[1] - vk[1], qz = vi[2] - vk[2];
    double q = sqrt(qx * qx + qy * qy + qz * qz);
    acc = vhs_accept(X->P, &X->sigma, q, xa, &X->st->violations);
  }
  if (acc) {
    orc_collide_pair(vi, vk, xi1, xi2);
    X->vx[si] = vi[0]; X->vy[si] = vi[1]; X->vz[si] = vi[2];
    X->vx[sk] = vk[0]; X->vy[sk] = vk[1]; X->vz[sk] = vk[2];
    X->st->accepted += 1;
  }
  log_coll(X->lg, X->K.gcell, r, d, j, si, sk, acc);
}

/* ===================================================================== */
/* Alg 4.3 / 4.4 in level-synchronous (LS) form [R2, R14, R17]             */
/* Level d collisions: C_d = ceil((N_d + cons_d)/2) (repeat...until N_n>0, */
/* "N_n = N_n - 2"); each draws k uniform in {0..d-1}            */
/* and consumes one sample of f_k and one of f_{d-1-k}; samples of */
/* f_0 are original particles, samples of f_k, k>=1, are outputs   */
/* of level-k collisions ("stored particles").                  */
/* ===================================================================== */
typedef struct {
  int64_t C; int32_t *type; int64_t *slot;
  double *len;            /* TRMC-WB: tree length of each collision's outputs        */
  unsigned char *used;    /* TRMC-WB: output o consumed by a higher level (2C flags) */
} level_t;

/* TRMC-WB (sec. 4.4, eqs def:1-3): length of a sample of f_k made by a
 * collision of samples of f_j and f_h (k = h + j + 1) with lengths a, b. */
static double wb_combine(int32_t def, int32_t k, double a, double b) {
  if (def == 1) return 1.0 + (a < b ? a : b);        /* eq. (def:2) */
  if (def == 2) return 1.0 + 0.5 * (a + b);          /* eq. (def:3) */
  return (double)k;                                  /* eq. (def:1) */
}

/* Alg 4.5 on an explicit path list (the pin of Table 1). */
static double tree_len_rec(const int32_t *path, int64_t len, int64_t *pos, int32_t k, int32_t def,
                           int *bad) {
  if (k == 0) return 0.0;
  if (*pos + 2 > len) { *bad = 1; return 0.0; }
  const int32_t j = path[(*pos)++], h = path[(*pos)++];
  if (j < 0 || h < 0 || j + h + 1 != k) { *bad = 1; return 0.0; }
  const double a = tree_len_rec(path, len, pos, j, def, bad);
  const double b = tree_len_rec(path, len, pos, h, def, bad);
  return wb_combine(def, k, a, b);
}

double orc_tree_length(const int32_t *path, int64_t len, int32_t def, int64_t *used) {
  if (len < 1) { if (used) *used = -1; return 0.0; }
  int64_t pos = 1;
  int bad = 0;
  const double L = tree_len_rec(path, len, &pos, path[0], def, &bad);
  if (used) *used = bad ? -1 : pos;
  return L;
}

typedef struct {
  int32_t top;      /* highest level planned (0: nothing) */
  int64_t L;        /* leaves consumed = cons_0            */
  level_t *lv;      /* lv[1..top]                           */
  int32_t nlv;
} plan_t;

static void plan_free(plan_t *pl) {
  if (!pl->lv) return;
  for (int d = 0; d < pl->nlv; d++) {
    free(pl->lv[d].type); free(pl->lv[d].slot); free(pl->lv[d].len); free(pl->lv[d].used);
  }
  free(pl->lv);
  pl->lv = NULL;
}

/* Top-down counts for attempt r over levels 1..hi; quotas N[d] only for
 * lo <= d <= hi.  Feasibility guard (finite N bounds the tree):
 * while the leaves needed exceed `budget`, drop the top quota level. */
static void plan_counts(const keyctx *K, int r, int32_t lo, int32_t hi, const int64_t *N,
                        int64_t budget, plan_t *pl) {
  int32_t top = hi;
  while (top >= lo && N[top] == 0) top--;
  pl->nlv = (hi > 0 ? hi : 0) + 1;
  pl->lv = (level_t *)calloc((size_t)pl->nlv, sizeof(level_t));
  int64_t *cons = (int64_t *)calloc((size_t)pl->nlv, sizeof(int64_t));
  for (;;) {
    if (top < lo || top < 1) { pl->top = 0; pl->L = 0; break; }
    for (int d = 0; d <= top; d++) cons[d] = 0;
    for (int d = top; d >= 1; d--) {
      int64_t Q = (d >= lo) ? N[d] : 0;
      int64_t C = (Q + cons[d] + 1) / 2;
      free(pl->lv[d].type);
      pl->lv[d].C = C;
      pl->lv[d].type = (int32_t *)malloc(sizeof(int32_t) * (size_t)(C > 0 ? C : 1));
      for (int64_t j = 0; j < C; j++) {
        uint32_t w[4];
        draw(K, ORC_P_TYPE, r, d, (uint32_t)j, w);
        int32_t a = (int32_t)(((uint64_t)w[0] * (uint64_t)d) >> 32);  /* uniform in {0..d-1} */
        pl->lv[d].type[j] = a;
        cons[a] += 1;
        cons[d - 1 - a] += 1;
      }
    }
    if (cons[0] <= budget) { pl->top = top; pl->L = cons[0]; break; }
    for (int d = 1; d <= top; d++) pl->lv[d].C = 0;   /* guard: drop the top level */
    top--;
    while (top >= lo && N[top] == 0) top--;
  }
  free(cons);
}

/* Bottom-up: resolve each collision's two input slots, then execute it.
 * Demands on pool p are ranked, within level d, side-0 demands (type p) in
 * j order then side-1 demands (type d-1-p) in j order; pool p's k-th demand
 * overall takes output pi_p(k) of level p (pi_0: the cell's leaf order). */
static void plan_execute(cellctx *X, int r, plan_t *pl, const uint32_t rk0[4], int64_t n,
                         int64_t leaf_off) {
  int32_t top = pl->top;
  if (top < 1) return;
  int64_t *base = (int64_t *)calloc((size_t)top + 1, sizeof(int64_t));
  int64_t *cnt = (int64_t *)calloc((size_t)top + 1, sizeof(int64_t));
  uint32_t (*rk)[4] = calloc((size_t)top + 1, sizeof *rk);
  for (int p = 1; p <= top; p++) draw(&X->K, ORC_P_PERM, r, p, 0, rk[p]);
  for (int d = 1; d <= top; d++) {
    level_t *L = &pl->lv[d];
    int64_t C = L->C;
    if (C == 0) continue;
    int64_t *rank = (int64_t *)malloc(sizeof(int64_t) * (size_t)C);
    for (int64_t j = 0; j < C; j++) rank[j] = cnt[L->type[j]]++;
    L->slot = (int64_t *)malloc(sizeof(int64_t) * 2 * (size_t)C);
    L->len = (double *)calloc((size_t)C, sizeof(double));
    L->used = (unsigned char *)calloc(2 * (size_t)C, 1);
    for (int64_t j = 0; j < C; j++) {
      int32_t a = L->type[j], b = d - 1 - a;
      int64_t t[2] = {base[a] + rank[j], base[b] + cnt[b] + rank[j]};
      int32_t pool[2] = {a, b};
      double in_len[2] = {0.0, 0.0};            /* samples of f_0 have length 0 */
      for (int s = 0; s < 2; s++) {
        if (pool[s] == 0) {
          L->slot[2 * j + s] = orc_feistel((uint64_t)(leaf_off + t[s]), (uint64_t)n, rk0);
        } else {
          level_t *Lp = &pl->lv[pool[s]];
          int64_t o = orc_feistel((uint64_t)t[s], (uint64_t)(2 * Lp->C), rk[pool[s]]);
          L->slot[2 * j + s] = Lp->slot[o];
          Lp->used[o] = 1;
          in_len[s] = Lp->len[o / 2];
        }
      }
      L->len[j] = wb_combine(X->P->wb, d, in_len[0], in_len[1]);
    }
    for (int p = 0; p < d; p++) base[p] += cnt[p] + cnt[d - 1 - p];
    for (int64_t j = 0; j < C; j++) cnt[L->type[j]] = 0;
    free(rank);
    for (int64_t j = 0; j < C; j++)
      tree_collision(X, r, d, j, L->slot[2 * j], L->slot[2 * j + 1]);
  }
  free(base); free(cnt); free(rk);
}

/* ===================================================================== */
/* Literal recursive Alg 4.3 / 4.4 (statistical cross-check only, [R2]).  */
/* ===================================================================== */
typedef struct {
  cellctx *X; const uint32_t *rk0; int64_t n, leaf; int err;
  int64_t *Nk; int64_t **store; int64_t *cnt; int64_t *capst;
  uint32_t ctr; double buf[2]; int nbuf; int64_t nodes;
} literal_t;

static double lit_uniform(literal_t *T) {
  if (T->nbuf == 0) {
    uint32_t w[4];
    draw(&T->X->K, ORC_P_LITERAL, 0, 0, T->ctr++, w);
    T->buf[0] = orc_u53(w[0], w[1]);
    T->buf[1] = orc_u53(w[2], w[3]);
    T->nbuf = 2;
  }
  return T->buf[--T->nbuf];
}

static void lit_sample(literal_t *T, int lev, int64_t *oi, int64_t *oj);

static int64_t lit_get(literal_t *T, int k) {
  if (k == 0) {                                         /* "take v_i from f_0" */
    if (T->leaf >= T->n) { T->err = 1; return 0; }
    return orc_feistel((uint64_t)T->leaf++, (uint64_t)T->n, T->rk0);
  }
  if (T->cnt[k] > 0) {                                  /* stored particle, random choice */
    int64_t idx = (int64_t)(lit_uniform(T) * (double)T->cnt[k]);
    int64_t s = T->store[k][idx];
    T->store[k][idx] = T->store[k][--T->cnt[k]];
    T->Nk[k] += 1;
    return s;
  }
  int64_t a, b;                                         /* sample v_i, v_i* recursively */
  lit_sample(T, k, &a, &b);
  if (T->cnt[k] == T->capst[k]) {
    T->capst[k] = T->capst[k] ? 2 * T->capst[k] : 8;
    T->store[k] = (int64_t *)realloc(T->store[k], sizeof(int64_t) * (size_t)T->capst[k]);
  }
  T->store[k][T->cnt[k]++] = b;
  T->Nk[k] -= 1;
  return a;
}

static void lit_sample(literal_t *T, int lev, int64_t *oi, int64_t *oj) {
  int k = (int)(lit_uniform(T) * (double)lev);          /* k uniform in {0..lev-1} */
  int64_t i = lit_get(T, k);
  int64_t j = lit_get(T, lev - k - 1);
  cellctx *X = T->X;
  double vi[3] = {X->vx[i], X->vy[i], X->vz[i]}, vj[3] = {X->vx[j], X->vy[j], X->vz[j]};
  int acc = 1;
  double xa = lit_uniform(T), xi1 = lit_uniform(T), xi2 = lit_uniform(T);
  X->st->proposals += 1;
  if (X->P->model != ORC_MAXWELL) {
    double qx = vi[0] - vj[0], qy = vi[1] - vj[1], qz = vi[2] - vj[2];
    double q = sqrt(qx * qx + qy * qy + qz * qz);
    acc = vhs_accept(X->P, &X->sigma, q, xa, &X->st->violations);
  }
  if (acc) {
    orc_collide_pair(vi, vj, xi1, xi2);
    X->vx[i] = vi[0]; X->vy[i] = vi[1]; X->vz[i] = vi[2];
    X->vx[j] = vj[0]; X->vy[j] = vj[1]; X->vz[j] = vj[2];
    X->st->accepted += 1;
  }
  T->nodes++;
  *oi = i; *oj = j;
}

/* ===================================================================== */
/* One cell: A3 moments/majorant, A4 split, A5-A6 trees, A7 RAD, A8 Max.  */
/* ===================================================================== */
static int cmp_i64(const void *a, const void *b) {
  int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
  return (x > y) - (x < y);
}

/* indicator of the post-collision state with Theta taken analytically
 * (P:646-649): Pxx (default [R20]) or M4. */
static double rad_estimate(cellctx *X, int64_t n, const unsigned char *inTheta,
                           const int64_t *theta, int64_t nT, double ux, double uy, double uz) {
  double s = 0;
  for (int64_t i = 0; i < n; i++) {
    if (inTheta[i]) continue;
    if (X->P->indicator == ORC_IND_PXX) {
      double dx = X->vx[i] - ux;
      s += dx * dx;
    } else {
      double v2 = X->vx[i] * X->vx[i] + X->vy[i] * X->vy[i] + X->vz[i] * X->vz[i];
      s += v2 * v2;
    }
  }
  if (nT > 0) {
    double tx = 0, ty = 0, tz = 0;
    for (int64_t q = 0; q < nT; q++) { tx += X->vx[theta[q]]; ty += X->vy[theta[q]]; tz += X->vz[theta[q]]; }
    tx /= (double)nT; ty /= (double)nT; tz /= (double)nT;
    double e = 0;
    for (int64_t q = 0; q < nT; q++) {
      double dx = X->vx[theta[q]] - tx, dy = X->vy[theta[q]] - ty, dz = X->vz[theta[q]] - tz;
      e += dx * dx + dy * dy + dz * dz;
    }
    double T = e / (3.0 * (double)nT);
    if (X->P->indicator == ORC_IND_PXX) {
      s += (double)nT * (T + (tx - ux) * (tx - ux));
    } else {
      double u2 = tx * tx + ty * ty + tz * tz;
      s += (double)nT * (u2 * u2 + 10.0 * u2 * T + 15.0 * T * T);
    }
  }
  return s / (double)n;
}

static int collide_cell(const orc_params *P, keyctx K, double rho_c, int64_t n, double *vx,
                        double *vy, double *vz, int32_t *m_state, orc_cell_stats *st,
                        logger *lg) {
  memset(st, 0, sizeof *st);
  st->n = (double)n;
  int32_t m = P->adaptive ? *m_state : P->m_fixed;
  if (n == 0) { st->m_used = m; st->m_next = m; return 0; }

  /* A3: moments and majorant Sigma = sigma(2 dv) */
  double sx = 0, sy = 0, sz = 0;
  for (int64_t i = 0; i < n; i++) { sx += vx[i]; sy += vy[i]; sz += vz[i]; }
  double ux = sx / (double)n, uy = sy / (double)n, uz = sz / (double)n;
  double dv2 = 0, pxx = 0, m4 = 0;
  for (int64_t i = 0; i < n; i++) {
    double dx = vx[i] - ux, dy = vy[i] - uy, dz = vz[i] - uz;
    double r2 = dx * dx + dy * dy + dz * dz;
    if (r2 > dv2) dv2 = r2;
    pxx += dx * dx;
    double v2 = vx[i] * vx[i] + vy[i] * vy[i] + vz[i] * vz[i];
    m4 += v2 * v2;
  }
  double S0 = (P->indicator == ORC_IND_PXX) ? pxx / (double)n : m4 / (double)n;
  double sigma = 0, mu;
  if (P->model == ORC_HARD_SPHERE) {
    sigma = 2.0 * sqrt(dv2);                    /* Sigma' = 2 dv; K = 1/(4 pi) [R4] */
    mu = rho_c * sigma;                         /* mu = 4 pi rho Sigma [R5]         */
  } else if (P->model == ORC_VHS) {
    sigma = pow(2.0 * sqrt(dv2), P->alpha);     /* Sigma' = sigma(2 dv) / K */
    mu = rho_c * sigma;
  } else {
    mu = rho_c;                                 /* Maxwell: mu = 4 pi rho K          */
  }
  double x = mu * P->dt / P->eps;
  double p = exp(-x);                           /* p = 1 - tau, tau of P:432        */
  st->p = p; st->mu = mu; st->sigma = sigma; st->S0 = S0;

  cellctx X = {P, K, sigma, vx, vy, vz, st, lg};
  uint32_t rk0[4];
  draw(&K, ORC_P_PERM, 0, 0, 0, rk0);           /* pi_0: order of f_0 particles */

  int32_t mmax = P->adaptive ? (P->m_cap > m ? P->m_cap : m) : m;
  int64_t *N = (int64_t *)calloc((size_t)mmax + 2, sizeof(int64_t));
  split_t sp;
  split_begin(&K, &sp, p, n, N);
  split_extend(&K, &sp, m, N);
  st->depth = sp.d;

  int rc = 0;
  if (P->literal) {
    /* literal Alg 4.3/4.4: for n = m..1 take N_n samples of f_n */
    literal_t T;
    memset(&T, 0, sizeof T);
    T.X = &X; T.rk0 = rk0; T.n = n;
    int32_t top = sp.d;
    T.Nk = (int64_t *)calloc((size_t)top + 1, sizeof(int64_t));
    T.store = (int64_t **)calloc((size_t)top + 1, sizeof(int64_t *));
    T.cnt = (int64_t *)calloc((size_t)top + 1, sizeof(int64_t));
    T.capst = (int64_t *)calloc((size_t)top + 1, sizeof(int64_t));
    for (int d = 0; d <= top; d++) T.Nk[d] = N[d];
    for (int lev = top; lev >= 1 && !T.err; lev--) {
      while (T.Nk[lev] > 0 && !T.err) {
        int64_t a, b;
        lit_sample(&T, lev, &a, &b);
        T.Nk[lev] -= 2;
      }
    }
    if (T.err) rc = -3;
    int64_t L = T.leaf;
    int64_t U = N[0] < n - L ? N[0] : n - L;
    int64_t nT = n - L - U;
    int64_t *theta = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nT > 0 ? nT : 1));
    for (int64_t q = 0; q < nT; q++) theta[q] = orc_feistel((uint64_t)(L + q), (uint64_t)n, rk0);
    qsort(theta, (size_t)nT, sizeof(int64_t), cmp_i64);
    orc_maxwellian(nT, theta, vx, vy, vz, K.seed, K.gcell, K.step);
    st->leaves = (double)L; st->untouched = (double)U; st->thermalised = (double)nT;
    st->maxw = nT >= 2 ? (double)nT : 0;
    st->m_used = m; st->m_next = m; st->attempts = 1;
    for (int d = 0; d <= top; d++) free(T.store[d]);
    free(T.Nk); free(T.store); free(T.cnt); free(T.capst); free(theta); free(N);
    return rc;
  }

  /* attempt 0: levels 1..d with quotas N_1..N_d, all n particles available */
  int r = 0;
  plan_t pl = {0};
  plan_counts(&K, r, 1, sp.d, N, n, &pl);
  plan_execute(&X, r, &pl, rk0, n, 0);
  /* TRMC-WB (Alg 4.6): final samples of f_d (outputs no higher
   * level consumed) whose tree is longer than wb_max join the Maxwellian set */
  int64_t nwb = 0;
  int64_t *wbs = NULL;
  if (P->wb && pl.top >= 1) {
    int64_t cap = 0;
    for (int d = 1; d <= pl.top; d++) cap += 2 * pl.lv[d].C;
    wbs = (int64_t *)malloc(sizeof(int64_t) * (size_t)(cap > 0 ? cap : 1));
    for (int d = 1; d <= pl.top; d++)
      for (int64_t o = 0; o < 2 * pl.lv[d].C; o++)
        if (!pl.lv[d].used[o] && pl.lv[d].len[o / 2] > (double)P->wb_max) wbs[nwb++] = pl.lv[d].slot[o];
  }
  plan_free(&pl);
  int64_t Ltot = pl.L;
  int64_t U = N[0] < n - Ltot ? N[0] : n - Ltot;
  int64_t nT = n - Ltot - U;

  unsigned char *inTheta = (unsigned char *)calloc((size_t)n, 1);
  int64_t *theta = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
  int32_t m_cur = m;
  double S_est = S0, E1 = 0;
  int32_t m_next = m;
  if (P->adaptive) {
    /* A7: TRMC-RAD, keep-and-extend on rejection [R22] */
    for (;;) {
      memset(inTheta, 0, (size_t)n);
      for (int64_t q = 0; q < nT; q++) {
        theta[q] = orc_feistel((uint64_t)(Ltot + q), (uint64_t)n, rk0);
        inTheta[theta[q]] = 1;
      }
      S_est = rad_estimate(&X, n, inTheta, theta, nT, ux, uy, uz);
      if (S0 != 0) E1 = fabs(S_est - S0) / fabs(S0);
      else E1 = (S_est == 0) ? 0.0 : INFINITY;
      if (E1 > P->delta2 && m_cur < P->m_cap) {
        int32_t m_new = 2 * m_cur < P->m_cap ? 2 * m_cur : P->m_cap;
        split_extend(&K, &sp, m_new, N);        /* continue the split: prefix property */
        r++;
        plan_t pr = {0};
        plan_counts(&K, r, m_cur + 1, sp.d, N, nT, &pr);   /* quotas only above m */
        plan_execute(&X, r, &pr, rk0, n, Ltot); /* leaves = next pi_0 positions in Theta */
        plan_free(&pr);
        Ltot += pr.L;
        nT -= pr.L;
        m_cur = m_new;
        continue;
      }
      break;
    }
    if (E1 < P->delta1) m_next = m_cur / 2 > 1 ? m_cur / 2 : 1;
    else m_next = m_cur;                        /* accept (or forced accept at m_cap) */
    *m_state = m_next;
  }
  st->depth = sp.d;

  /* A8: thermalised set Theta = pi_0 positions [Ltot, Ltot + nT) (plus the
   * TRMC-WB rejections), ascending slots */
  if (nwb > 0) theta = (int64_t *)realloc(theta, sizeof(int64_t) * (size_t)(n + nwb));
  for (int64_t q = 0; q < nT; q++) theta[q] = orc_feistel((uint64_t)(Ltot + q), (uint64_t)n, rk0);
  for (int64_t q = 0; q < nwb; q++) theta[nT + q] = wbs[q];
  qsort(theta, (size_t)(nT + nwb), sizeof(int64_t), cmp_i64);
  orc_maxwellian(nT + nwb, theta, vx, vy, vz, K.seed, K.gcell, K.step);
  free(wbs);

  st->S_est = S_est; st->E1 = E1;
  st->m_used = m_cur; st->m_next = m_next; st->attempts = r + 1;
  st->leaves = (double)Ltot; st->untouched = (double)U; st->thermalised = (double)nT;
  st->maxw = nT + nwb >= 2 ? (double)(nT + nwb) : 0;
  free(inTheta); free(theta); free(N);
  return rc;
}

int32_t orc_step_cells(const orc_params *P, int64_t ncells, const int64_t *offsets,
                       uint32_t gcell0, const double *rho, uint32_t step,
                       double *vx, double *vy, double *vz, int32_t *m_state,
                       orc_cell_stats *stats, orc_coll_rec *log, int64_t log_cap,
                       int64_t *log_n) {
  logger lg = {log, log_cap, 0};
  int32_t rc = 0;
  for (int64_t c = 0; c < ncells; c++) {
    keyctx K = {P->seed, gcell0 + (uint32_t)c, step};
    int64_t o = offsets[c], n = offsets[c + 1] - offsets[c];
    int r = collide_cell(P, K, rho ? rho[c] : 1.0, n, vx + o, vy + o, vz + o, m_state + c,
                         &stats[c], log ? &lg : NULL);
    if (r) rc = r;
  }
  if (log_n) *log_n = lg.n;
  return rc;
}

/* ===================================================================== */
/* A9: per-cell moments                             */
/* ===================================================================== */
void orc_moments(int64_t ncells, const int64_t *offsets, const double *rho, const double *vx,
                 const double *vy, const double *vz, const int32_t *m_state, double *out) {
  for (int64_t c = 0; c < ncells; c++) {
    int64_t o = offsets[c], n = offsets[c + 1] - offsets[c];
    double *r = out + 12 * c;
    memset(r, 0, 12 * sizeof(double));
    r[0] = (double)n;
    r[1] = rho ? rho[c] : 1.0;
    r[11] = m_state ? (double)m_state[c] : 0.0;
    if (n == 0) continue;
    double sx = 0, sy = 0, sz = 0;
    for (int64_t i = o; i < o + n; i++) { sx += vx[i]; sy += vy[i]; sz += vz[i]; }
    double ux = sx / (double)n, uy = sy / (double)n, uz = sz / (double)n;
    double e = 0, pxx = 0, m4 = 0, m4c = 0;
    for (int64_t i = o; i < o + n; i++) {
      double dx = vx[i] - ux, dy = vy[i] - uy, dz = vz[i] - uz;
      double c2 = dx * dx + dy * dy + dz * dz;
      double v2 = vx[i] * vx[i] + vy[i] * vy[i] + vz[i] * vz[i];
      e += c2; pxx += dx * dx; m4 += v2 * v2; m4c += c2 * c2;
    }
    double T = e / (3.0 * (double)n);
    r[2] = ux; r[3] = uy; r[4] = uz; r[5] = T;
    r[6] = 0.5 * r[1] * (ux * ux + uy * uy + uz * uz + 3.0 * T);   /* E = 3/2 rho T + 1/2 rho u^2 */
    r[7] = r[1] * T;                                                 /* p = rho T */
    r[8] = pxx / (double)n; r[9] = m4 / (double)n; r[10] = m4c / (double)n;
  }
}

/* ===================================================================== */
/* 1D stationary shock: reservoirs (A1), transport (A1), stable sort (A2)  */
/* ===================================================================== */
int32_t orc_rankine_hugoniot(double mach, double gamma, double rho_L, double T_L, double out[6]) {
  if (!(mach > 1.0) || !(gamma > 1.0) || !(rho_L > 0) || !(T_L > 0)) return -1;
  /* rho_L u_L = rho_R u_R; rho_L u_L^2 + p_L = rho_R u_R^2 + p_R;
   * u_L (E_L + p_L) = u_R (E_R + p_R), p = rho T.               */
  double M2 = mach * mach;
  double u_L = mach * sqrt(gamma * T_L);
  double rho_R = rho_L * (gamma + 1.0) * M2 / ((gamma - 1.0) * M2 + 2.0);
  double p_R = rho_L * T_L * (2.0 * gamma * M2 - (gamma - 1.0)) / (gamma + 1.0);
  double u_R = rho_L * u_L / rho_R;
  out[0] = rho_L; out[1] = u_L; out[2] = T_L;
  out[3] = rho_R; out[4] = u_R; out[5] = p_R / rho_R;
  return 0;
}

static int32_t cell_of(const orc_shock *S, double x) {
  double inv = (double)S->ncells / (S->x_max - S->x_min);
  double f = floor((x - S->x_min) * inv);
  int32_t c = (f < 0) ? 0 : (f >= (double)S->ncells ? S->ncells - 1 : (int32_t)f);
  return c;
}

/* stable counting sort of the sequence (src order) by cell */
static void stable_bin(const orc_shock *S, int64_t m, const int32_t *cell, const double *x,
                       const double *vx, const double *vy, const double *vz, double *ox,
                       double *ovx, double *ovy, double *ovz, int64_t *offsets) {
  int32_t C = S->ncells;
  for (int32_t c = 0; c <= C; c++) offsets[c] = 0;
  for (int64_t i = 0; i < m; i++) offsets[cell[i] + 1]++;
  for (int32_t c = 0; c < C; c++) offsets[c + 1] += offsets[c];
  int64_t *pos = (int64_t *)malloc(sizeof(int64_t) * (size_t)C);
  for (int32_t c = 0; c < C; c++) pos[c] = offsets[c];
  for (int64_t i = 0; i < m; i++) {
    int64_t k = pos[cell[i]]++;
    ox[k] = x[i]; ovx[k] = vx[i]; ovy[k] = vy[i]; ovz[k] = vz[i];
  }
  free(pos);
}

int32_t orc_shock_bin(const orc_shock *S, int64_t n, double *x, double *vx, double *vy,
                      double *vz, int64_t *offsets) {
  int32_t *cell = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  for (int64_t i = 0; i < n; i++) {
    if (!(x[i] >= S->x_min && x[i] < S->x_max)) { free(cell); return -1; }
    cell[i] = cell_of(S, x[i]);
  }
  size_t b = sizeof(double) * (size_t)(n > 0 ? n : 1);
  double *ox = malloc(b), *ovx = malloc(b), *ovy = malloc(b), *ovz = malloc(b);
  stable_bin(S, n, cell, x, vx, vy, vz, ox, ovx, ovy, ovz, offsets);
  memcpy(x, ox, sizeof(double) * (size_t)n); memcpy(vx, ovx, sizeof(double) * (size_t)n);
  memcpy(vy, ovy, sizeof(double) * (size_t)n); memcpy(vz, ovz, sizeof(double) * (size_t)n);
  free(ox); free(ovx); free(ovy); free(ovz); free(cell);
  return 0;
}

int32_t orc_shock_step(const orc_params *P, const orc_shock *S, uint32_t step, int64_t *n_io,
                       int64_t cap, double *x, double *vx, double *vy, double *vz,
                       int64_t *offsets, int32_t *m_state, orc_cell_stats *stats,
                       double *counts_out) {
  int64_t n = *n_io;
  int32_t C = S->ncells;
  double dx = (S->x_max - S->x_min) / (double)C;
  /* A1 reservoirs: ghost slabs of width Lg = (|u_B| + 6 sqrt(T_B)) dt refilled
   * with IR(rho_B Lg / w) particles of M(rho_B, u_B, T_B) at uniform positions. */
  int64_t ng[2] = {0, 0};
  double *gx[2], *gv[2][3];
  for (int side = 0; side < 2; side++) {
    double rhoB = side ? S->rho_R : S->rho_L, uB = side ? S->u_R : S->u_L;
    double TB = side ? S->T_R : S->T_L;
    double Lg = (fabs(uB) + 6.0 * sqrt(TB)) * P->dt;
    keyctx K = {P->seed, 0xFFFFFFF0u + (uint32_t)side, step};
    uint32_t w[4];
    draw(&K, ORC_P_RESV, side, 0, 0, w);
    ng[side] = orc_ir(rhoB * Lg / S->weight, orc_u53(w[0], w[1]));
    size_t b = sizeof(double) * (size_t)(ng[side] > 0 ? ng[side] : 1);
    gx[side] = malloc(b);
    for (int k = 0; k < 3; k++) gv[side][k] = malloc(b);
    double sT = sqrt(TB);
    for (int64_t k = 0; k < ng[side]; k++) {
      uint32_t a[4], bb[4], cc[4];
      draw(&K, ORC_P_RESV, side, 1, (uint32_t)k, a);
      draw(&K, ORC_P_RESV, side, 2, (uint32_t)k, bb);
      draw(&K, ORC_P_RESV, side, 3, (uint32_t)k, cc);
      double upos = orc_u53(a[0], a[1]), u1 = orc_u53(a[2], a[3]);
      double u2 = orc_u53(bb[0], bb[1]), u3 = orc_u53(bb[2], bb[3]), u4 = orc_u53(cc[0], cc[1]);
      gx[side][k] = side ? S->x_max + Lg * upos : (S->x_min - Lg) + Lg * upos;
      double r1 = sqrt(-2.0 * log(u1)), r3 = sqrt(-2.0 * log(u3));
      gv[side][0][k] = uB + sT * (r1 * cos(2.0 * M_PI * u2));
      gv[side][1][k] = sT * (r1 * sin(2.0 * M_PI * u2));
      gv[side][2][k] = sT * (r3 * cos(2.0 * M_PI * u4));
    }
  }
  /* A1 transport x <- x + v_x dt, A2 stable sort by destination.
   * Canonical source order: left ghosts, interior particles, right ghosts. */
  int64_t tot = ng[0] + n + ng[1];
  size_t b = sizeof(double) * (size_t)(tot > 0 ? tot : 1);
  double *sx = malloc(b), *svx = malloc(b), *svy = malloc(b), *svz = malloc(b);
  int32_t *cell = malloc(sizeof(int32_t) * (size_t)(tot > 0 ? tot : 1));
  int64_t m = 0, dropped = 0, inj[2] = {0, 0};
  for (int part = 0; part < 3; part++) {
    int64_t cnt = part == 1 ? n : ng[part == 0 ? 0 : 1];
    for (int64_t i = 0; i < cnt; i++) {
      double px, pvx, pvy, pvz;
      if (part == 1) { px = x[i]; pvx = vx[i]; pvy = vy[i]; pvz = vz[i]; }
      else {
        int sd = part == 0 ? 0 : 1;
        px = gx[sd][i]; pvx = gv[sd][0][i]; pvy = gv[sd][1][i]; pvz = gv[sd][2][i];
      }
      double xn = px + pvx * P->dt;
      if (!(xn >= S->x_min && xn < S->x_max)) { if (part == 1) dropped++; continue; }
      if (part != 1) inj[part == 0 ? 0 : 1]++;
      sx[m] = xn; svx[m] = pvx; svy[m] = pvy; svz[m] = pvz; cell[m] = cell_of(S, xn);
      m++;
    }
  }
  for (int side = 0; side < 2; side++) { free(gx[side]); for (int k = 0; k < 3; k++) free(gv[side][k]); }
  if (m > cap) { free(sx); free(svx); free(svy); free(svz); free(cell); return -2; }
  stable_bin(S, m, cell, sx, svx, svy, svz, x, vx, vy, vz, offsets);
  free(sx); free(svx); free(svy); free(svz); free(cell);
  *n_io = m;
  if (counts_out) {
    counts_out[0] = (double)inj[0]; counts_out[1] = (double)inj[1];
    counts_out[2] = (double)dropped; counts_out[3] = (double)(ng[0] + ng[1]);
  }
  /* A3-A8 per cell with rho_c = n_c w / dx */
  int32_t rc = 0;
  for (int32_t c = 0; c < C; c++) {
    keyctx K = {P->seed, (uint32_t)c, step};
    int64_t o = offsets[c], nc = offsets[c + 1] - offsets[c];
    double rho_c = (double)nc * S->weight / dx;
    int r = collide_cell(P, K, rho_c, nc, vx + o, vy + o, vz + o, m_state + c, &stats[c], NULL);
    if (r) rc = r;
  }
  return rc;
}
