// fused.cuh — the fused shock step (A1 transport + A2 sort + A3-A8 collisions in
// one pass over the particles; DESIGN.md §5 "fused shock step").
//
// The legacy step streams the state three times (transport_kernel: read x, v_x,
// write x and a destination; scatter_sorted: read and write (x, v); the
// collision kernel: read v, write v) - 68 B per fp32 particle against the 32 B
// minimum of SURVEY 8(d) D3 (read and write (x, v) once).  The fused step keeps
// the same canonical state (cell-sorted arrays, canonical order inside a cell,
// DESIGN.md §3.3) plus a 1-byte "move code" per particle, computed by the
// kernel that finishes the particle's cell: where the particle's NEXT transport
// takes it (same cell S, left neighbour L, right neighbour R, dropped D, or
// farther F - listed separately).  With the codes, the destination cell d of
// the next step is, in canonical source order,
//     [left ghosts][left immigrants][far movers from cells < d-1]
//     [R of cell d-1][S of cell d][L of cell d+1]
//     [far movers from cells > d+1][right immigrants][right ghosts],
// each part in slot order - exactly the stable counting sort of the oracle
// (stable_bin), so the fp64 results are bitwise those of the legacy path.
// One warp per destination cell gathers that list from the source buffer
// (transporting on the fly: x' = x + v_x dt, the legacy arithmetic), places it
// at the cell's final offset in the destination buffer, runs the collision
// step in place (cell_warp.cuh phases) and writes the codes of the particles'
// next move.  The offsets come from the per-cell code counts (fused_counts +
// the scan) before the pass.  Per particle this reads (x, v) and writes (x, v)
// and one code byte: 33 B.
#pragma once

namespace trmcr {

enum : int8_t { kCodeS = 0, kCodeL = 1, kCodeR = 2, kCodeF = 3, kCodeD = 4 };

// Per-buffer-parity side data of the fused step (parity = the buffer it describes).
struct FusedDev {
  int8_t *code[2];              // [cap] move code of each particle of buffer b
  int32_t *nlsr[2];             // [3 C] per cell: L, S, R counts of buffer b
  int32_t *far_src[2];          // [far_cap] index in buffer b of a far mover
  int32_t *far_dst[2];          // [far_cap] its local destination cell
  int *far_cnt;                 // [2]
  int far_cap;
};

// Move codes of cell c (n particles at [base, base + n) of buffer par, positions
// x after this step's transport, final velocities): the next transport
// x'' = x + v_x dt with the legacy arithmetic (cell = floor((x'' - x_min) / dx),
// tested against the three candidate cells first).  Warp-cooperative.
template <typename Real>
__device__ void warp_codes(const ShockDev &S, const FusedDev &F, int par, int c, int64_t base, int n,
                           const Real *__restrict__ xs, const Real *__restrict__ vxs, int *err) {
  constexpr int U = 4;
  const int lane = threadIdx.x & 31;
  const Real *__restrict__ xb = xs + base;
  const Real *__restrict__ vb = vxs + base;
  int8_t *__restrict__ code_out = F.code[par] + base;
  const double g = (double)(c + S.cbase);            // this cell's global index (exact)
  int nl = 0, nr = 0, nd = 0;
  for (int i0 = 0; i0 < n; i0 += 32 * U) {
    Real xv[U], vv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u * 32 + lane;
      xv[u] = i < n ? xb[i] : Real(0);
      vv[u] = i < n ? vb[i] : Real(0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u * 32 + lane;
      if (i >= n) continue;
      const Real xn = add_rn<Real>(xv[u], mul_rn<Real>(vv[u], (Real)S.dt));
      const double xd = (double)xn;
      int8_t code;
      if (!(xd >= S.x_min && xd < S.x_max)) {
        code = kCodeD;
      } else {
        const double f = (xd - S.x_min) * S.inv_dx;     // cell_of's argument of floor
        if (f >= g && f < g + 1.0) code = kCodeS;
        else if (f >= g - 1.0 && f < g && c > 0) code = kCodeL;
        else if (f >= g + 1.0 && f < g + 2.0 && c + 1 < S.C) code = kCodeR;
        else {
          const int d = cell_of(S, xd) - S.cbase;
          if (d == c) code = kCodeS;                   // clamped at the domain's last cell
          else if (d == c - 1) code = kCodeL;
          else if (d == c + 1) code = kCodeR;
          else {
            code = kCodeF;
            if (d < 0 || d >= S.C) {
              atomicOr(err, 32);                     // more than one cell into a neighbouring slab
            } else {
              const int k = atomicAdd(&F.far_cnt[par], 1);
              if (k < F.far_cap) { F.far_src[par][k] = (int32_t)(base + i); F.far_dst[par][k] = d; }
              else atomicOr(err, 128);               // far-mover list full
            }
          }
        }
      }
      code_out[i] = code;
      nl += code == kCodeL;
      nr += code == kCodeR;
      nd += code >= kCodeF;
    }
  }
  nl = __reduce_add_sync(0xffffffffu, nl);
  nr = __reduce_add_sync(0xffffffffu, nr);
  nd = __reduce_add_sync(0xffffffffu, nd);
  if (lane == 0) {
    int32_t *r = F.nlsr[par] + 3 * (size_t)c;
    r[0] = nl; r[1] = n - nl - nr - nd; r[2] = nr;
  }
}

// Codes of every cell of buffer c->cur (after init / set_particles /
// set_velocities, or after a legacy step): one warp per cell.
template <typename Real>
__global__ void __launch_bounds__(256) codes_kernel(ShockDev S, FusedDev F, int par, const int64_t *__restrict__ off,
                                                    const Real *x, const Real *vx, int *err) {
  pdl_wait();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int c = warp; c < S.C; c += nw) {
    const int64_t b = off[c];
    warp_codes<Real>(S, F, par, c, b, (int)(off[c + 1] - b), x, vx, err);
  }
  pdl_trigger();
}

// counts[d] (ghosts, immigrants, far movers: added before) += R(d-1) + S(d) + L(d+1).
__global__ void __launch_bounds__(256) fused_counts(ShockDev S, const int32_t *__restrict__ nlsr, int32_t *counts) {
  pdl_wait();
  for (int d = blockIdx.x * blockDim.x + threadIdx.x; d < S.C; d += gridDim.x * blockDim.x) {
    int k = nlsr[3 * (size_t)d + 1];
    if (d > 0) k += nlsr[3 * (size_t)(d - 1) + 2];
    if (d + 1 < S.C) k += nlsr[3 * (size_t)(d + 1)];
    counts[d] += k;
  }
  pdl_trigger();
}

// far movers of the previous step join the destination counts (one CTA).
__global__ void __launch_bounds__(256) far_count(const FusedDev F, int par, int32_t *counts, int *W) {
  pdl_wait();
  const int nf = min(F.far_cnt[par], F.far_cap);
  for (int k = threadIdx.x; k < nf; k += blockDim.x) atomicAdd(&counts[F.far_dst[par][k]], 1);
  pdl_trigger();
}

// Append one source segment to the warp's output: lanes with `take` set, in lane
// order after `pos`.  Returns the new pos.
template <typename Real>
__device__ __forceinline__ int put_lane(bool take, int pos, Real x, Real vx, Real vy, Real vz, Real *ox, Real *ovx,
                                        Real *ovy, Real *ovz, int cap) {
  const int lane = threadIdx.x & 31;
  const unsigned m = __ballot_sync(0xffffffffu, take);
  if (take) {
    const int q = pos + __popc(m & ((1u << lane) - 1u));
    if (q < cap) { ox[q] = x; ovx[q] = vx; ovy[q] = vy; ovz[q] = vz; }
  }
  return pos + __popc(m);
}

// Interior particles of source cell s with move code `want`, in slot order,
// transported (x' = x + v_x dt), appended at out[pos...].  Each lane takes W
// consecutive slots (one 16-byte vector per array, W = 4 floats or 2 doubles;
// the codes as one W-byte word), a warp scan of the per-lane counts gives the
// output positions (the source and destination buffers never alias).
template <typename Real>
__device__ __forceinline__ int gather_coded(const ShockDev &S, const GatherSrc &G, const FusedDev &F, int par, int s,
                                            int8_t want, int pos, Real *__restrict__ ox, Real *__restrict__ ovx,
                                            Real *__restrict__ ovy, Real *__restrict__ ovz, int cap) {
  using V = typename Vec<Real>::T;
  constexpr int Wv = Vec<Real>::W;
  const int lane = threadIdx.x & 31;
  const int lo = (int)G.off_old[s], hi = (int)G.off_old[s + 1];
  if (hi <= lo) return pos;
  const int8_t *__restrict__ code = F.code[par];
  const Real *__restrict__ x = (const Real *)G.x;
  const Real *__restrict__ vx = (const Real *)G.vx;
  const Real *__restrict__ vy = (const Real *)G.vy;
  const Real *__restrict__ vz = (const Real *)G.vz;
  const Real dt = (Real)S.dt;
  const uint32_t wmask = want * (Wv == 4 ? 0x01010101u : 0x0101u);
  for (int a0 = lo - lo % Wv; a0 < hi; a0 += 32 * Wv) {
    const int a = a0 + lane * Wv;
    unsigned bits = 0;
    if (a < hi) {
      uint32_t cw;
      if constexpr (Wv == 4) cw = *reinterpret_cast<const uint32_t *>(code + a);
      else cw = *reinterpret_cast<const uint16_t *>(code + a);
      cw ^= wmask;                                     // byte k == 0  <=>  code[a + k] == want
#pragma unroll
      for (int k = 0; k < Wv; ++k)
        if (((cw >> (8 * k)) & 0xFFu) == 0u && a + k >= lo && a + k < hi) bits |= 1u << k;
    }
    const int cnt = __popc(bits);
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    if (bits) {
      const V xv = *reinterpret_cast<const V *>(x + a), bv = *reinterpret_cast<const V *>(vx + a);
      const V cv = *reinterpret_cast<const V *>(vy + a), dv = *reinterpret_cast<const V *>(vz + a);
      int q = pos + incl - cnt;
#pragma unroll
      for (int k = 0; k < Wv; ++k) {
        if ((bits >> k) & 1u) {
          if (q < cap) {
            const Real b = vget<V, Real>(bv, k);
            ox[q] = add_rn<Real>(vget<V, Real>(xv, k), mul_rn<Real>(b, dt));
            ovx[q] = b; ovy[q] = vget<V, Real>(cv, k); ovz[q] = vget<V, Real>(dv, k);
          }
          ++q;
        }
      }
    }
    pos += total;
  }
  return pos;
}

// Far movers (previous step's list) with destination c from source cells
// before (before = true: below c - 1) or after c + 1, in source order.  The list
// is in arbitrary order: every match is ranked by counting the matches with a
// smaller source index (the list is empty or tiny at CFL < 1).
template <typename Real>
__device__ int gather_far(const ShockDev &S, const GatherSrc &G, const FusedDev &F, int par, int c, bool before,
                          int pos, Real *ox, Real *ovx, Real *ovy, Real *ovz, int cap) {
  const int lane = threadIdx.x & 31;
  const int nf = min(F.far_cnt[par], F.far_cap);
  if (nf == 0) return pos;
  const int64_t cut = before ? G.off_old[max(c - 1, 0)] : G.off_old[min(c + 2, S.C)];
  const int32_t *fs = F.far_src[par], *fd = F.far_dst[par];
  auto match = [&](int k) { return fd[k] == c && (before ? fs[k] < cut : fs[k] >= cut); };
  const Real *x = (const Real *)G.x, *vx = (const Real *)G.vx, *vy = (const Real *)G.vy, *vz = (const Real *)G.vz;
  int total = 0;
  for (int k0 = 0; k0 < nf; k0 += 32) {
    const int k = k0 + lane;
    const bool m = k < nf && match(k);
    if (m) {
      const int32_t src = fs[k];
      int rank = 0;
      for (int j = 0; j < nf; ++j) rank += (match(j) && fs[j] < src) ? 1 : 0;
      const int q = pos + rank;
      if (q < cap) {
        const Real b = vx[src];
        ox[q] = add_rn<Real>(x[src], mul_rn<Real>(b, (Real)S.dt));
        ovx[q] = b; ovy[q] = vy[src]; ovz[q] = vz[src];
      }
    }
    total += __popc(__ballot_sync(0xffffffffu, m));
  }
  return pos + total;
}

// Already-transported particles (reservoir ghosts of one side, or immigrants)
// whose destination equals `match`, in index order.
template <typename Real>
__device__ __forceinline__ int gather_list(int cnt, const Real *px, const Real *pvx, const Real *pvy,
                                           const Real *pvz, const int32_t *pd, int match, int pos, Real *ox,
                                           Real *ovx, Real *ovy, Real *ovz, int cap) {
  const int lane = threadIdx.x & 31;
  for (int k0 = 0; k0 < cnt; k0 += 32) {
    const int k = k0 + lane;
    const bool take = k < cnt && pd[k] == match;
    Real a = Real(0), b = Real(0), cc = Real(0), d = Real(0);
    if (take) { a = px[k]; b = pvx[k]; cc = pvy[k]; d = pvz[k]; }
    pos = put_lane<Real>(take, pos, a, b, cc, d, ox, ovx, ovy, ovz, cap);
  }
  return pos;
}

// The particles of destination cell c in canonical order, placed at out
// (ox..ovz already offset to the cell's first slot).  Returns the count.
template <typename Real>
__device__ int gather_fused_warp(const ShockDev &S, const GatherSrc &G, const FusedDev &F, int par, int c, Real *ox,
                                 Real *ovx, Real *ovy, Real *ovz, int cap) {
  const int W = *G.W;     // reach of ghosts / immigrants from the domain or slab edges
  int pos = 0;
  const bool left_edge = c - W <= -1, right_edge = c + W >= S.C;
  if (left_edge) {
    pos = gather_list<Real>(G.ng[0], (const Real *)G.gx[0], (const Real *)G.gvx[0], (const Real *)G.gvy[0],
                            (const Real *)G.gvz[0], G.gdest[0], c, pos, ox, ovx, ovy, ovz, cap);
    if (G.recv[0]) {
      const XBuf<Real> X = XBuf<Real>::bind(const_cast<void *>(G.recv[0]), G.xcap);
      pos = gather_list<Real>(min(*X.count, G.xcap), X.x, X.vx, X.vy, X.vz, X.dest, c + G.cbase, pos, ox, ovx, ovy,
                              ovz, cap);
    }
  }
  pos = gather_far<Real>(S, G, F, par, c, true, pos, ox, ovx, ovy, ovz, cap);
  if (c > 0) pos = gather_coded<Real>(S, G, F, par, c - 1, kCodeR, pos, ox, ovx, ovy, ovz, cap);
  pos = gather_coded<Real>(S, G, F, par, c, kCodeS, pos, ox, ovx, ovy, ovz, cap);
  if (c + 1 < S.C) pos = gather_coded<Real>(S, G, F, par, c + 1, kCodeL, pos, ox, ovx, ovy, ovz, cap);
  pos = gather_far<Real>(S, G, F, par, c, false, pos, ox, ovx, ovy, ovz, cap);
  if (right_edge) {
    if (G.recv[1]) {
      const XBuf<Real> X = XBuf<Real>::bind(const_cast<void *>(G.recv[1]), G.xcap);
      pos = gather_list<Real>(min(*X.count, G.xcap), X.x, X.vx, X.vy, X.vz, X.dest, c + G.cbase, pos, ox, ovx, ovy,
                              ovz, cap);
    }
    pos = gather_list<Real>(G.ng[1], (const Real *)G.gx[1], (const Real *)G.gvx[1], (const Real *)G.gvy[1],
                            (const Real *)G.gvz[1], G.gdest[1], c, pos, ox, ovx, ovy, ovz, cap);
  }
  __syncwarp();
  return pos;
}

// Slab exchange in fused mode: the emigrants are the L-coded particles of cell 0
// (to the left slab) and the R-coded ones of cell C-1 (to the right), in slot
// order, transported; a far mover into a neighbouring slab is an error (32,
// flagged by warp_codes).  One warp per side.
template <typename Real>
__global__ void __launch_bounds__(32) pack_emigrants_fused(ShockDev S, GatherSrc G, FusedDev F, int par,
                                                           void *send_l, void *send_r, int cap, int *err) {
  pdl_wait();
  const int side = blockIdx.x, lane = threadIdx.x;
  if (side == 0 ? !S.has_left : !S.has_right) { pdl_trigger(); return; }
  XBuf<Real> B = XBuf<Real>::bind(side == 0 ? send_l : send_r, cap);
  const int s = side == 0 ? 0 : S.C - 1;
  const int8_t want = side == 0 ? kCodeL : kCodeR;
  const int gdest = S.cbase + (side == 0 ? -1 : S.C);
  const int64_t lo = G.off_old[s], hi = G.off_old[s + 1];
  const Real *x = (const Real *)G.x, *vx = (const Real *)G.vx, *vy = (const Real *)G.vy, *vz = (const Real *)G.vz;
  int pos = 0;
  for (int64_t i0 = lo; i0 < hi; i0 += 32) {
    const int64_t i = i0 + lane;
    const bool take = i < hi && F.code[par][i] == want;
    const unsigned m = __ballot_sync(0xffffffffu, take);
    if (take) {
      const int q = pos + __popc(m & ((1u << lane) - 1u));
      if (q < cap) {
        const Real b = vx[i];
        B.x[q] = add_rn<Real>(x[i], mul_rn<Real>(b, (Real)S.dt));
        B.vx[q] = b; B.vy[q] = vy[i]; B.vz[q] = vz[i]; B.dest[q] = gdest;
      }
    }
    pos += __popc(m);
  }
  if (lane == 0) {
    if (pos > cap) { atomicOr(err, 2); pos = cap; }
    *B.count = pos;
  }
  pdl_trigger();
}

// Bulk L2 prefetch (TMA engine, no registers or completion tracking) of a byte
// range, widened to 16-byte alignment.
__device__ __forceinline__ void prefetch_l2(const void *p, size_t bytes) {
  uintptr_t a = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15);
  const uintptr_t e = (reinterpret_cast<uintptr_t>(p) + bytes + 15) & ~uintptr_t(15);
  while (a < e) {
    const uint32_t sz = (uint32_t)((e - a) < (uintptr_t(1) << 16) ? (e - a) : (uintptr_t(1) << 16));
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(sz) : "memory");
    a += sz;
  }
}

// The source range of the cells [c0 - 1, c0 + kLockWarps] (what a lock group's
// gathers read) into L2: one lane per array.
template <typename Real>
__device__ __forceinline__ void prefetch_group(const ShockDev &S, const GatherSrc &G, const FusedDev &F, int par,
                                               int c0) {
  const int lane = threadIdx.x & 31;
  if (c0 >= S.C || lane >= 5) return;
  const int64_t lo = G.off_old[max(c0 - 1, 0)], hi = G.off_old[min(c0 + kLockWarps + 1, S.C)];
  if (hi <= lo) return;
  if (lane == 4) { prefetch_l2(F.code[par] + lo, (size_t)(hi - lo)); return; }
  const void *arr[4] = {G.x, G.vx, G.vy, G.vz};
  prefetch_l2((const Real *)arr[lane] + lo, (size_t)(hi - lo) * sizeof(Real));
}

// The fused pass (lock-step groups as shock_collide_lock): per destination cell,
// gather + transport into place, collision step in place, move codes.
template <typename Real, bool WB>
__global__ void __launch_bounds__(kLockWarps * 32, 16 / kLockWarps)
shock_fused_lock(StepParams P, WarpSlabLayout Lay, ShockDev S, GatherSrc G, FusedDev F, int par_in,
                 const int64_t *__restrict__ off_new, Real *ox, Real *ovx, Real *ovy, Real *ovz, int32_t *m_state,
                 double *stats, int *defer_count, int *defer_list, QueueArgs Q) {
  pdl_wait();
  if (off_new[S.C] > S.cap) { pdl_trigger(); return; }   // capacity exceeded (err set by the scan): no stores
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int par_out = par_in ^ 1;
  unsigned char *slab = smem + (size_t)warp * Lay.per_warp;
  WarpShared &sh = *reinterpret_cast<WarpShared *>(slab + Lay.off_sh);
  CellBuf<Real> B;
  double *usplit;
  bind_warp_slab(B, slab, Lay, usplit);
  for (int base = blockIdx.x * kLockWarps; base < S.C; base += gridDim.x * kLockWarps) {
    const int c = base + warp;
    int64_t b0 = 0;
    int n = 0, rc = kOk;
    bool run = false;
    if (c < S.C) {
      b0 = off_new[c];
      n = (int)(off_new[c + 1] - b0);
      const int got = gather_fused_warp<Real>(S, G, F, par_in, c, ox + b0, ovx + b0, ovy + b0, ovz + b0, n);
      if (got != n && lane == 0) atomicOr(Q.err, kErrInternal);
      B.vx = ovx + b0; B.vy = ovy + b0; B.vz = ovz + b0;
      if (n > Lay.n_cap) {
        rc = kOverflow;
      } else if (n == 0) {
        if (lane == 0) {
          double *st = stats + (size_t)c * TRMCR_NSTATS;
          for (int k = 0; k < TRMCR_NSTATS; ++k) st[k] = 0.0;
          const int m = P.adaptive ? m_state[c] : P.m_fixed;
          st[TRMCR_ST_MUSED] = m; st[TRMCR_ST_MNEXT] = m;
          int32_t *r = F.nlsr[par_out] + 3 * (size_t)c;
          r[0] = 0; r[1] = 0; r[2] = 0;
        }
      } else {
        double sx = 0, sy = 0, sz = 0;
        if constexpr (sizeof(Real) == 4) {
          float fx = 0, fy = 0, fz = 0;
          for (int i = lane; i < n; i += 32) { fx += B.vx[i]; fy += B.vy[i]; fz += B.vz[i]; }
          sx = fx; sy = fy; sz = fz;
        } else {
          for (int i = lane; i < n; i += 32) { sx += B.vx[i]; sy += B.vy[i]; sz += B.vz[i]; }
        }
        rc = wphase_begin<Real>(P, B, sh, usplit, sx, sy, sz, n, P.cell_base + (uint32_t)c, m_state + c);
        run = rc == kOk;
      }
    }
    const bool work = run;
    __syncthreads();
    while (run) {
      rc = wphase_attempt<Real, WB>(P, B, sh, usplit, P.cell_base + (uint32_t)c, Q.log, Q.log_count, Q.log_cap);
      run = rc == kOk && !sh.done;
    }
    if (work && rc == kOk) {
      wphase_end<Real, WB>(P, B, sh, B.vx, B.vy, B.vz, P.cell_base + (uint32_t)c, m_state + c,
                           stats + (size_t)c * TRMCR_NSTATS);
      __syncwarp();
      warp_codes<Real>(S, F, par_out, c, b0, n, ox, ovx, Q.err);
    }
    if (c < S.C && rc != kOk && lane == 0) defer_list[atomicAdd(defer_count, 1)] = c;
    __syncthreads();
  }
  pdl_trigger();
}

}  // namespace trmcr
