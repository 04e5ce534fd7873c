/*
 * trmcr_oracle.h — TEST INFRASTRUCTURE ONLY (see trmcr_oracle.c header).
 *
 * Plain single-threaded CPU oracle of the TRMC-R hot path, arXiv:1009.2768.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it.  It shares no code with paper_1009_2768_b200/ (the product path).
 */
#ifndef TRMCR_ORACLE_H
#define TRMCR_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_MAXWELL = 0, ORC_HARD_SPHERE = 1, ORC_VHS = 2 };   /* B = K|q|^alpha, alpha = 0, 1, or in (0,1) */
enum { ORC_IND_PXX = 0, ORC_IND_M4 = 1 };

/* Philox purposes. */
enum {
  ORC_P_SPLIT = 1, ORC_P_TYPE = 2, ORC_P_PERM = 3, ORC_P_COLL = 4, ORC_P_COLL2 = 5,
  ORC_P_MAXW = 6, ORC_P_MAXW2 = 7, ORC_P_RESV = 8, ORC_P_RESV2 = 9, ORC_P_LITERAL = 10
};

typedef struct {
  int32_t model;       /* ORC_MAXWELL | ORC_HARD_SPHERE                         */
  int32_t adaptive;    /* 0: fixed m (TRMC-R, Alg 4.4); 1: TRMC-RAD (§4.3)      */
  int32_t m_fixed;     /* truncation order when adaptive == 0                   */
  int32_t m_init;      /* initial m_max (RAD)                                   */
  int32_t m_cap;       /* largest m_max (RAD)                                   */
  int32_t indicator;   /* ORC_IND_PXX | ORC_IND_M4                              */
  double delta1, delta2;
  double eps, dt;
  uint64_t seed;
  int32_t literal;     /* 1: literal recursive Alg 4.3/4.4 (statistical checks) */
  int32_t pad;
  double alpha;        /* ORC_VHS exponent                          */
  int32_t wb;          /* TRMC-WB tree length (sec. 4.4): 0 off, 1 eq.(def:2)   */
                       /* 1 + min, 2 eq.(def:3) 1 + mean, 3 eq.(def:1) = level  */
  int32_t wb_max;      /* m_max of Alg 4.6: final samples with L > wb_max are   */
                       /* resampled from the local Maxwellian                   */
  int32_t sigma_update;/* 1: majorant raised to sigma_ij after each proposal    */
                       /* (remark after Alg 4.4); 0: frozen per step */
} orc_params;

/* Length of one collision tree given as the path list of Alg 4.5:
 * path[0] = k; for k > 0 the list continues j, h, then the sub-list of f_j,
 * then the sub-list of f_h (each sub-list without its own leading k).
 * def = 1 (1 + min), 2 (1 + mean), 3 (the coefficient k, eq. def:1).
 * Returns the length; *used = entries read (negative on a malformed list). */
double orc_tree_length(const int32_t *path, int64_t len, int32_t def, int64_t *used);

/* Per-cell result of one collision step (all counts as doubles for ctypes). */
typedef struct {
  double n;            /* particles in the cell                                 */
  double p;            /* e^{-mu dt/eps}  (= 1 - tau)                            */
  double mu;           /* majorant rate                                         */
  double sigma;        /* Sigma' = 2 sqrt(max|v - u|^2)  (HS), 0 for Maxwell     */
  double S0;           /* indicator before the step                             */
  double S_est;        /* indicator estimate of the accepted attempt            */
  double E1;           /* |S_est - S0| / |S0| of the accepted attempt           */
  double m_used;       /* m of the accepted attempt                             */
  double m_next;       /* m_max for the next step                               */
  double depth;        /* realised split depth m'                               */
  double attempts;     /* 1 + number of RAD retries                             */
  double leaves;       /* L: particles consumed as f_0 leaves                   */
  double untouched;    /* U                                                      */
  double thermalised;  /* |Theta|                                                */
  double proposals;    /* collisions (tree nodes), dummy included                */
  double accepted;     /* accepted collisions                                   */
  double violations;   /* pairs with |q|^a > Sigma' (1 + 2^-40) [R35]           */
  double maxw;         /* Maxwellian samples drawn                               */
} orc_cell_stats;

/* One record per tree node (collision) for decision parity. */
typedef struct {
  int32_t cell;        /* global cell id                                         */
  int32_t attempt;
  int32_t level;       /* d                                                      */
  int32_t accepted;
  int64_t j;           /* index within the level                                 */
  int64_t slot_i, slot_k;
} orc_coll_rec;

/* ---- primitives (exported for unit pins) ---- */
void    orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
double  orc_u53(uint32_t hi, uint32_t lo);
int64_t orc_ir(double y, double u);
int64_t orc_feistel(uint64_t x, uint64_t N, const uint32_t rk[4]);
void    orc_collide_pair(double *vi, double *vj, double xi1, double xi2);
int32_t orc_split(double p, int64_t n, int32_t m, uint64_t seed, uint32_t gcell, uint32_t step,
                  int64_t *N_out /* [m+2] */, int64_t *rem_out);
void    orc_maxwellian(int64_t k, const int64_t *slots, double *vx, double *vy, double *vz,
                       uint64_t seed, uint32_t gcell, uint32_t step);

/* ---- one collision step on homogeneous cells (in place, fp64) ----
 * cells are [offsets[c], offsets[c+1]); global id gcell0 + c; density rho[c].
 * m_state[c] is RAD's m_max (in/out).  log may be NULL; *log_n counts records
 * (records beyond log_cap are counted but not written). Returns 0 or <0 error. */
int32_t orc_step_cells(const orc_params *P, int64_t ncells, const int64_t *offsets,
                       uint32_t gcell0, const double *rho, uint32_t step,
                       double *vx, double *vy, double *vz, int32_t *m_state,
                       orc_cell_stats *stats, orc_coll_rec *log, int64_t log_cap,
                       int64_t *log_n);

/* ---- per-cell moments (A9): 12 doubles per cell ----
 * [n, rho, ux, uy, uz, T, E, pressure, Pxx, M4, M4c, m_max] */
void orc_moments(int64_t ncells, const int64_t *offsets, const double *rho,
                 const double *vx, const double *vy, const double *vz,
                 const int32_t *m_state, double *out);

/* ---- 1D shock (A1, A2) ---- */
typedef struct {
  int32_t ncells;      /* C                                                      */
  int32_t pad;
  double x_min, x_max; /* domain                                                 */
  double weight;       /* mass per particle w                                    */
  double rho_L, u_L, T_L, rho_R, u_R, T_R;  /* reservoir states                  */
} orc_shock;

/* Transport + reservoirs + stable counting sort (A1, A2), then per-cell
 * collision step.  Particles are SoA (x, vx, vy, vz) of length *n, sorted by
 * cell, offsets[C+1] describes them; arrays have capacity cap.  In/out. */
int32_t orc_shock_step(const orc_params *P, const orc_shock *S, uint32_t step,
                       int64_t *n, int64_t cap, double *x, double *vx, double *vy, double *vz,
                       int64_t *offsets, int32_t *m_state, orc_cell_stats *stats,
                       double *counts_out /* [4]: injected L, injected R, dropped, far */);

/* Stable bin of unsorted particles by cell (used at init): reorders in place. */
int32_t orc_shock_bin(const orc_shock *S, int64_t n, double *x, double *vx, double *vy,
                      double *vz, int64_t *offsets);

/* Rankine-Hugoniot right state for a monatomic-gamma gas (§5.2). */
int32_t orc_rankine_hugoniot(double mach, double gamma, double rho_L, double T_L,
                             double out[6] /* rho_L,u_L,T_L,rho_R,u_R,T_R */);

#ifdef __cplusplus
}
#endif
#endif
