// comm.cuh — the multi-GPU surface of the library: an NCCL
// communicator per context, created from a unique id that the caller moves
// between processes (torch.distributed broadcasts the 128 bytes), and the three
// collectives of the path, all on the context's streams:
//   * global moments of independent cells: all-reduce of the 10 sums on a
//     communication stream, overlapped with the next step (P:829-832 cost and
//     moments, configs[2]);
//   * the 1D shock's neighbour exchange between trmcr_shock_begin and
//     trmcr_shock_finish: one ncclSend/ncclRecv pair per neighbour in one group
//     (fixed-capacity buffers with a count header: no size round trip);
//   * partition-independent global results: all-gather of the per-cell rows,
//     summed on the host with an exactly rounded sum (Shewchuk's algorithm, as
//     math.fsum), so the totals are bitwise the same for any number of GPUs.
#pragma once
#include <nccl.h>

#include <cmath>

#include "ctx.cuh"

namespace trmcr {

#define NCCL_TRY(ctx, call)                                                                   \
  do {                                                                                        \
    ncclResult_t r_ = (call);                                                                 \
    if (r_ != ncclSuccess) {                                                                  \
      (ctx)->sticky = 1;                                                                      \
      return fail(ctx, TRMCR_ENCCL, std::string(#call " failed: ") + ncclGetErrorString(r_)); \
    }                                                                                         \
  } while (0)

// Exactly rounded sum of doubles (Shewchuk 1997 / Python's math.fsum): the
// partials are non-overlapping and their exact sum is the exact sum of the
// inputs; the last step rounds it once (half-even).  Finite inputs only.
inline double exact_sum(const double *v, size_t n, size_t stride) {
  std::vector<double> p;
  p.reserve(32);
  for (size_t k = 0; k < n; ++k) {
    double x = v[k * stride];
    size_t i = 0;
    for (double y : p) {
      if (std::fabs(x) < std::fabs(y)) std::swap(x, y);
      const double hi = x + y;
      const double lo = y - (hi - x);
      if (lo != 0.0) p[i++] = lo;
      x = hi;
    }
    p.resize(i);
    p.push_back(x);
  }
  if (p.empty()) return 0.0;
  size_t i = p.size() - 1;
  double hi = p[i], lo = 0.0;
  while (i > 0) {
    const double x = hi, y = p[--i];
    hi = x + y;
    const double yr = hi - x;
    lo = y - yr;
    if (lo != 0.0) break;
  }
  // half-even correction: the remaining partials decide a tie
  if (i > 0 && ((lo < 0.0 && p[i - 1] < 0.0) || (lo > 0.0 && p[i - 1] > 0.0))) {
    const double y = lo * 2.0, x = hi + y;
    if (y == x - hi) hi = x;
  }
  return hi;
}

inline trmcr_status comm_init(trmcr_ctx *c, const void *nccl_id, int rank, int nranks) {
  c->rank = rank;
  c->nranks = nranks;
  if (!nccl_id) return nranks == 1 ? TRMCR_OK : fail(c, TRMCR_EINVAL, "nranks > 1 needs an NCCL unique id");
  ncclUniqueId id;
  memcpy(&id, nccl_id, sizeof(id));
  NCCL_TRY(c, ncclCommInitRank(&c->comm, nranks, id, rank));
  CUDA_TRY(c, cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking));
  CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_comm_ready, cudaEventDisableTiming));
  for (int k = 0; k < kCommSlots; ++k) CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_comm_done[k], cudaEventDisableTiming));
  if (c->geometry == TRMCR_SHOCK_1D) {
    ShockState &s = c->shock;
    if (s.has_left != (rank > 0) || s.has_right != (rank + 1 < nranks))
      return fail(c, TRMCR_EINVAL, "shock slabs: rank r must own the r-th slab (neighbours = ranks r-1, r+1)");
    if (s.has_left || s.has_right) {   // the library's own exchange buffers
      CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_pack, cudaEventDisableTiming));
      CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_xchg, cudaEventDisableTiming));
      const int cap = 1 << 13;
      const size_t b = c->dtype == TRMCR_F64 ? XBuf<double>::bytes(cap) : XBuf<float>::bytes(cap);
      void *buf[4] = {nullptr, nullptr, nullptr, nullptr};
      for (int k = 0; k < 4; ++k) {
        if (dalloc(c, &buf[k], b)) return TRMCR_ENOMEM;
        CUDA_TRY(c, cudaMemsetAsync(buf[k], 0, b, c->stream));
      }
      s.xsend[0] = s.has_left ? buf[0] : nullptr; s.xsend[1] = s.has_right ? buf[1] : nullptr;
      s.xrecv[0] = s.has_left ? buf[2] : nullptr; s.xrecv[1] = s.has_right ? buf[3] : nullptr;
      s.xcap = cap;
      s.xbytes = b;
      s.own_xbuf = 1;
    }
  }
  return TRMCR_OK;
}

inline void comm_destroy(trmcr_ctx *c) {
  if (c->comm) ncclCommDestroy(c->comm);
  if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
  if (c->ev_comm_ready) cudaEventDestroy(c->ev_comm_ready);
  if (c->ev_pack) cudaEventDestroy(c->ev_pack);
  if (c->ev_xchg) cudaEventDestroy(c->ev_xchg);
  for (int k = 0; k < kCommSlots; ++k)
    if (c->ev_comm_done[k]) cudaEventDestroy(c->ev_comm_done[k]);
}

// Neighbour exchange of a shock slab (between shock_begin and shock_finish):
// send_left -> rank - 1 (its recv_right), send_right -> rank + 1 (its
// recv_left).  The whole fixed-capacity buffer travels.  It runs on the
// communication stream, after the event shock_begin recorded behind the pack
// kernel, so it overlaps the bulk transport that shock_begin launched after
// the pack; the context stream resumes (immigrant counts, offsets, sort,
// collisions) when the exchange is done.
inline trmcr_status comm_shock_exchange(trmcr_ctx *c) {
  ShockState &s = c->shock;
  const size_t b = s.xbytes;
  cudaStream_t xs = c->ev_pack && c->ev_xchg && c->comm_stream ? c->comm_stream : c->stream;
  if (xs != c->stream) CUDA_TRY(c, cudaStreamWaitEvent(xs, c->ev_pack, 0));
  NCCL_TRY(c, ncclGroupStart());
  if (s.has_left) {
    NCCL_TRY(c, ncclSend(s.xsend[0], b, ncclUint8, c->rank - 1, c->comm, xs));
    NCCL_TRY(c, ncclRecv(s.xrecv[0], b, ncclUint8, c->rank - 1, c->comm, xs));
  }
  if (s.has_right) {
    NCCL_TRY(c, ncclSend(s.xsend[1], b, ncclUint8, c->rank + 1, c->comm, xs));
    NCCL_TRY(c, ncclRecv(s.xrecv[1], b, ncclUint8, c->rank + 1, c->comm, xs));
  }
  NCCL_TRY(c, ncclGroupEnd());
  if (xs != c->stream) {
    CUDA_TRY(c, cudaEventRecord(c->ev_xchg, xs));
    CUDA_TRY(c, cudaStreamWaitEvent(c->stream, c->ev_xchg, 0));
  }
  return TRMCR_OK;
}

// Slot of a caller's global-moments buffer: its all-reduce's completion event.
inline int comm_slot(trmcr_ctx *c, const void *p) {
  for (int k = 0; k < kCommSlots; ++k)
    if (c->comm_ptr[k] == p) return k;
  const int k = c->comm_next;
  c->comm_next = (c->comm_next + 1) % kCommSlots;
  c->comm_ptr[k] = p;
  return k;
}

// All ranks' per-cell rows (k doubles per cell), in global cell order, on the
// host of every rank.  Synchronises.
inline trmcr_status comm_allgather_rows(trmcr_ctx *c, const double *dev_rows, int k, std::vector<double> &out,
                                        int64_t &cells_total) {
  if (!c->comm) {
    out.resize((size_t)c->ncells * k);
    CUDA_TRY(c, cudaMemcpyAsync(out.data(), dev_rows, sizeof(double) * out.size(), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    cells_total = c->ncells;
    return TRMCR_OK;
  }
  const int R = c->nranks;
  // (cell_base, ncells) of every rank
  int64_t *d_meta = nullptr;
  if (dalloc(c, &d_meta, sizeof(int64_t) * 2 * (R + 1))) return TRMCR_ENOMEM;
  const int64_t mine[2] = {c->cell_base, c->ncells};
  CUDA_TRY(c, cudaMemcpyAsync(d_meta + 2 * R, mine, sizeof(mine), cudaMemcpyHostToDevice, c->stream));
  NCCL_TRY(c, ncclAllGather(d_meta + 2 * R, d_meta, 2, ncclInt64, c->comm, c->stream));
  std::vector<int64_t> meta(2 * R);
  CUDA_TRY(c, cudaMemcpyAsync(meta.data(), d_meta, sizeof(int64_t) * 2 * R, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  int64_t maxc = 0;
  cells_total = 0;
  for (int r = 0; r < R; ++r) { maxc = std::max(maxc, meta[2 * r + 1]); cells_total += meta[2 * r + 1]; }
  const size_t per = (size_t)std::max<int64_t>(maxc, 1) * k;
  double *d_send = nullptr, *d_all = nullptr;
  if (dalloc(c, &d_send, sizeof(double) * per) || dalloc(c, &d_all, sizeof(double) * per * R)) return TRMCR_ENOMEM;
  CUDA_TRY(c, cudaMemsetAsync(d_send, 0, sizeof(double) * per, c->stream));
  if (c->ncells > 0)
    CUDA_TRY(c, cudaMemcpyAsync(d_send, dev_rows, sizeof(double) * (size_t)c->ncells * k, cudaMemcpyDeviceToDevice,
                                c->stream));
  NCCL_TRY(c, ncclAllGather(d_send, d_all, per, ncclDouble, c->comm, c->stream));
  std::vector<double> all(per * R);
  CUDA_TRY(c, cudaMemcpyAsync(all.data(), d_all, sizeof(double) * all.size(), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  for (void *p : {(void *)d_meta, (void *)d_send, (void *)d_all}) {   // one-shot buffers
    c->allocs.erase(std::remove(c->allocs.begin(), c->allocs.end(), p), c->allocs.end());
    cudaFree(p);
  }
  // assemble in global cell order (ranks sorted by cell_base)
  std::vector<int> order(R);
  for (int r = 0; r < R; ++r) order[r] = r;
  std::sort(order.begin(), order.end(), [&](int a, int b) { return meta[2 * a] < meta[2 * b]; });
  out.clear();
  out.reserve((size_t)cells_total * k);
  for (int r : order) out.insert(out.end(), all.begin() + per * r, all.begin() + per * r + meta[2 * r + 1] * k);
  return TRMCR_OK;
}

}  // namespace trmcr
