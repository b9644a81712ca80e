// NCCL halo exchange and allreduces of libdg (see dg_comm.h).
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <condition_variable>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>

#include "dg_comm.h"

namespace dg {

// gather: buf[s][c][i] = field[elems[s] * estride + c * np + i]
__global__ void k_pack(const double* __restrict__ field, long long estride, int ncomp, int np,
                       const int* __restrict__ elems, int n, double* __restrict__ buf) {
  const long long tot = (long long)n * ncomp * np;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < tot; k += stride) {
    const long long s = k / ((long long)ncomp * np);
    const long long r = k - s * ncomp * np;
    buf[k] = field[(long long)elems[s] * estride + r];
  }
}

// scatter received ghosts into rows [n_el, n_tot) of a strided field
__global__ void k_unpack(double* __restrict__ field, long long estride, int ncomp, int np,
                         int n_el, int n_ghost, const double* __restrict__ buf) {
  const long long tot = (long long)n_ghost * ncomp * np;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < tot; k += stride) {
    const long long s = k / ((long long)ncomp * np);
    const long long r = k - s * ncomp * np;
    field[(long long)(n_el + s) * estride + r] = buf[k];
  }
}

// face-row plans: buf[k] = field[idx[k]] and field[idx[k]] = buf[k]
__global__ void k_pack_idx(const double* __restrict__ field, const long long* __restrict__ idx,
                           long long n, double* __restrict__ buf) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride)
    buf[k] = field[idx[k]];
}
__global__ void k_unpack_idx(double* __restrict__ field, const long long* __restrict__ idx,
                             long long n, const double* __restrict__ buf) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride)
    field[idx[k]] = buf[k];
}

#define NCCK(call)                                                    \
  do {                                                                \
    ncclResult_t _r = (call);                                         \
    if (_r != ncclSuccess) {                                          \
      err_ = std::string(#call) + ": " + ncclGetErrorString(_r);      \
      return false;                                                   \
    }                                                                 \
  } while (0)

#define CUCK(call)                                                    \
  do {                                                                \
    cudaError_t _e = (call);                                          \
    if (_e != cudaSuccess) {                                          \
      err_ = std::string(#call) + ": " + cudaGetErrorString(_e);      \
      return false;                                                   \
    }                                                                 \
  } while (0)

bool Comm::unique_id(void* out128, std::string* err) {
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) {
    if (err) *err = std::string("ncclGetUniqueId: ") + ncclGetErrorString(r);
    return false;
  }
  static_assert(sizeof(ncclUniqueId) == 128, "unexpected ncclUniqueId size");
  std::memcpy(out128, &id, sizeof id);
  return true;
}

// ------------------------------------------------------------ loopback
struct LoopGroup {
  int n = 0;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  long long gen = 0;
  std::vector<const double*> sendbuf;
  std::vector<std::vector<int>> send_off;
  std::vector<std::vector<long long>> row_send_off[Comm::N_ROW_PLANS];
  std::vector<cudaEvent_t> ev_pack, ev_copied;
  std::vector<std::vector<double>> slots;
  std::vector<long long> n_el;
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    const long long g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

static std::mutex g_loop_mu;
static std::map<int, std::shared_ptr<LoopGroup>> g_loops;

bool Comm::init_plan(int rank, int nranks, const int32_t* send_counts, const int32_t* send_elems,
                     const int32_t* recv_counts, int n_el, int n_tot) {
  rank_ = rank;
  nranks_ = nranks;
  n_el_ = n_el;
  n_tot_ = n_tot;
  send_counts_.assign(send_counts, send_counts + nranks);
  recv_counts_.assign(recv_counts, recv_counts + nranks);
  send_off_.assign(nranks + 1, 0);
  recv_off_.assign(nranks + 1, 0);
  for (int p = 0; p < nranks; ++p) {
    send_off_[p + 1] = send_off_[p] + send_counts_[p];
    recv_off_[p + 1] = recv_off_[p] + recv_counts_[p];
  }
  n_send_ = send_off_[nranks];
  if (recv_off_[nranks] != n_tot - n_el) {
    err_ = "halo plan: received ghost count does not match n_tot - n_el";
    return false;
  }
  if (n_send_ > 0) {
    CUCK(cudaMalloc(&d_send_elems_, n_send_ * sizeof(int)));
    CUCK(cudaMemcpy(d_send_elems_, send_elems, n_send_ * sizeof(int), cudaMemcpyHostToDevice));
  }
  CUCK(cudaMalloc(&scratch_, 8 * sizeof(double) + nranks * sizeof(double)));
  return true;
}

bool Comm::init_loopback(int group, int rank, int nranks, const int32_t* send_counts,
                         const int32_t* send_elems, const int32_t* recv_counts, int n_el,
                         int n_tot) {
  if (nranks <= 1) {
    rank_ = 0;
    nranks_ = 1;
    return true;
  }
  std::shared_ptr<LoopGroup> G;
  {
    std::lock_guard<std::mutex> lk(g_loop_mu);
    auto& slot = g_loops[group];
    if (!slot) {
      slot = std::make_shared<LoopGroup>();
      slot->n = nranks;
      slot->sendbuf.assign(nranks, nullptr);
      slot->send_off.assign(nranks, {});
      for (auto& r : slot->row_send_off) r.assign(nranks, {});
      slot->ev_pack.assign(nranks, nullptr);
      slot->ev_copied.assign(nranks, nullptr);
      slot->slots.assign(nranks, {});
      slot->n_el.assign(nranks, 0);
    }
    if (slot->n != nranks) {
      err_ = "loopback group size mismatch";
      return false;
    }
    G = slot;
  }
  if (!init_plan(rank, nranks, send_counts, send_elems, recv_counts, n_el, n_tot)) return false;
  CUCK(cudaEventCreateWithFlags(&G->ev_pack[rank], cudaEventDisableTiming));
  CUCK(cudaEventCreateWithFlags(&G->ev_copied[rank], cudaEventDisableTiming));
  CUCK(cudaEventRecord(G->ev_copied[rank], 0));
  G->send_off[rank] = send_off_;
  G->n_el[rank] = n_el;
  loop_ = G.get();
  G->barrier();  // every rank registered
  offset_ = 0;
  for (int p = 0; p < rank; ++p) offset_ += G->n_el[p];
  // keep the group alive while any member uses it
  static std::mutex keep_mu;
  static std::vector<std::shared_ptr<LoopGroup>> keep;
  {
    std::lock_guard<std::mutex> lk(keep_mu);
    keep.push_back(G);
  }
  G->barrier();
  if (rank == 0) {
    std::lock_guard<std::mutex> lk(g_loop_mu);
    g_loops.erase(group);  // the id can be reused by a later group
  }
  return true;
}

bool Comm::ensure_bufs(size_t per) {
  return ensure_cap(std::max((size_t)n_send_, (size_t)(n_tot_ - n_el_)) * per);
}

bool Comm::ensure_cap(size_t need) {
  if (need > buf_cap_) {
    if (loop_) CUCK(cudaDeviceSynchronize());  // peers may still read the old buffer
    if (sendbuf_) cudaFree(sendbuf_);
    if (recvbuf_) cudaFree(recvbuf_);
    CUCK(cudaMalloc(&sendbuf_, need * sizeof(double)));
    CUCK(cudaMalloc(&recvbuf_, need * sizeof(double)));
    buf_cap_ = need;
  }
  return true;
}

// op: 0 sum, 1 max
bool Comm::loop_reduce(double* dev, int n, cudaStream_t st, int op) {
  LoopGroup* G = loop_;
  auto& mine = G->slots[rank_];
  if ((int)mine.size() < n) mine.resize(n);
  CUCK(cudaMemcpyAsync(mine.data(), dev, n * sizeof(double), cudaMemcpyDeviceToHost, st));
  CUCK(cudaStreamSynchronize(st));
  G->barrier();
  std::vector<double> r(G->slots[0].begin(), G->slots[0].begin() + n);
  for (int q = 1; q < G->n; ++q)
    for (int i = 0; i < n; ++i)
      r[i] = op == 0 ? r[i] + G->slots[q][i] : std::max(r[i], G->slots[q][i]);
  G->barrier();  // every rank has read the slots
  CUCK(cudaMemcpyAsync(dev, r.data(), n * sizeof(double), cudaMemcpyHostToDevice, st));
  CUCK(cudaStreamSynchronize(st));
  return true;
}

bool Comm::init(const void* uid, int rank, int nranks, const int32_t* send_counts,
                const int32_t* send_elems, const int32_t* recv_counts, int n_el, int n_tot) {
  rank_ = rank;
  nranks_ = nranks;
  n_el_ = n_el;
  n_tot_ = n_tot;
  if (nranks <= 1) return true;
  ncclUniqueId id;
  std::memcpy(&id, uid, sizeof id);
  ncclComm_t c;
  NCCK(ncclCommInitRank(&c, nranks, id, rank));
  comm_ = c;
  send_counts_.assign(send_counts, send_counts + nranks);
  recv_counts_.assign(recv_counts, recv_counts + nranks);
  send_off_.assign(nranks + 1, 0);
  recv_off_.assign(nranks + 1, 0);
  for (int p = 0; p < nranks; ++p) {
    send_off_[p + 1] = send_off_[p] + send_counts_[p];
    recv_off_[p + 1] = recv_off_[p] + recv_counts_[p];
  }
  n_send_ = send_off_[nranks];
  if (recv_off_[nranks] != n_tot - n_el) {
    err_ = "halo plan: received ghost count does not match n_tot - n_el";
    return false;
  }
  if (n_send_ > 0) {
    CUCK(cudaMalloc(&d_send_elems_, n_send_ * sizeof(int)));
    CUCK(cudaMemcpy(d_send_elems_, send_elems, n_send_ * sizeof(int), cudaMemcpyHostToDevice));
  }
  CUCK(cudaMalloc(&scratch_, 8 * sizeof(double) + nranks * sizeof(double)));
  // global element offset of this rank (owned ranges are contiguous in rank order)
  std::vector<double> counts(nranks, 0.0);
  counts[rank] = (double)n_el;
  double* dc = scratch_ + 8;
  CUCK(cudaMemcpy(dc, counts.data(), nranks * sizeof(double), cudaMemcpyHostToDevice));
  NCCK(ncclAllReduce(dc, dc, nranks, ncclDouble, ncclSum, c, 0));
  CUCK(cudaMemcpy(counts.data(), dc, nranks * sizeof(double), cudaMemcpyDeviceToHost));
  offset_ = 0;
  for (int p = 0; p < rank; ++p) offset_ += (long long)counts[p];
  return true;
}

bool Comm::exchange(double* field, int ncomp, int np, cudaStream_t st, long long estride) {
  if (nranks_ <= 1) return true;
  if (estride < 0) estride = (long long)ncomp * np;
  const size_t per = (size_t)ncomp * np;
  if (loop_) {
    LoopGroup* G = loop_;
    // the peers' copies out of our send buffer (previous exchange) are done
    for (int q = 0; q < nranks_; ++q)
      if (q != rank_) CUCK(cudaStreamWaitEvent(st, G->ev_copied[q], 0));
    if (!ensure_bufs(per)) return false;
    if (n_send_ > 0) {
      const long long tot = (long long)n_send_ * per;
      const int grid = (int)std::min<long long>((tot + 255) / 256, 4096);
      k_pack<<<grid, 256, 0, st>>>(field, estride, ncomp, np, d_send_elems_, n_send_, sendbuf_);
      CUCK(cudaGetLastError());
    }
    CUCK(cudaEventRecord(G->ev_pack[rank_], st));
    G->sendbuf[rank_] = sendbuf_;
    G->barrier();  // every rank's pack is recorded
    for (int q = 0; q < nranks_; ++q) {
      if (q == rank_ || recv_counts_[q] == 0) continue;
      CUCK(cudaStreamWaitEvent(st, G->ev_pack[q], 0));
      CUCK(cudaMemcpyAsync(recvbuf_ + (size_t)recv_off_[q] * per,
                           G->sendbuf[q] + (size_t)G->send_off[q][rank_] * per,
                           (size_t)recv_counts_[q] * per * sizeof(double), cudaMemcpyDeviceToDevice,
                           st));
    }
    CUCK(cudaEventRecord(G->ev_copied[rank_], st));
    G->barrier();  // every rank's copies are recorded
    const int ng = n_tot_ - n_el_;
    if (ng > 0) {
      const long long tot = (long long)ng * per;
      const int grid = (int)std::min<long long>((tot + 255) / 256, 4096);
      k_unpack<<<grid, 256, 0, st>>>(field, estride, ncomp, np, n_el_, ng, recvbuf_);
      CUCK(cudaGetLastError());
    }
    return true;
  }
  if (!ensure_bufs(per)) return false;
  if (n_send_ > 0) {
    const long long tot = (long long)n_send_ * per;
    const int grid = (int)std::min<long long>((tot + 255) / 256, 4096);
    k_pack<<<grid, 256, 0, st>>>(field, estride, ncomp, np, d_send_elems_, n_send_, sendbuf_);
    CUCK(cudaGetLastError());
  }
  ncclComm_t c = (ncclComm_t)comm_;
  NCCK(ncclGroupStart());
  for (int p = 0; p < nranks_; ++p) {
    if (p == rank_) continue;
    if (send_counts_[p] > 0)
      NCCK(ncclSend(sendbuf_ + (size_t)send_off_[p] * per, (size_t)send_counts_[p] * per,
                    ncclDouble, p, c, st));
    if (recv_counts_[p] > 0)
      NCCK(ncclRecv(recvbuf_ + (size_t)recv_off_[p] * per, (size_t)recv_counts_[p] * per,
                    ncclDouble, p, c, st));
  }
  NCCK(ncclGroupEnd());
  const int ng = n_tot_ - n_el_;
  if (ng > 0) {
    const long long tot = (long long)ng * per;
    const int grid = (int)std::min<long long>((tot + 255) / 256, 4096);
    k_unpack<<<grid, 256, 0, st>>>(field, estride, ncomp, np, n_el_, ng, recvbuf_);
    CUCK(cudaGetLastError());
  }
  return true;
}

bool Comm::set_rows(int which, const int64_t* send_counts, const int64_t* send_idx,
                    const int64_t* recv_counts, const int64_t* recv_idx) {
  if (which < 0 || which >= N_ROW_PLANS) {
    err_ = "face-row plan index out of range";
    return false;
  }
  if (nranks_ <= 1) return true;
  RowPlan& R = rows_[which];
  R.send_off.assign(nranks_ + 1, 0);
  R.recv_off.assign(nranks_ + 1, 0);
  for (int p = 0; p < nranks_; ++p) {
    R.send_off[p + 1] = R.send_off[p] + send_counts[p];
    R.recv_off[p + 1] = R.recv_off[p] + recv_counts[p];
  }
  R.n_send = R.send_off[nranks_];
  R.n_recv = R.recv_off[nranks_];
  if (R.d_send_idx) cudaFree(R.d_send_idx);
  if (R.d_recv_idx) cudaFree(R.d_recv_idx);
  R.d_send_idx = R.d_recv_idx = nullptr;
  if (R.n_send > 0) {
    CUCK(cudaMalloc(&R.d_send_idx, R.n_send * sizeof(long long)));
    CUCK(cudaMemcpy(R.d_send_idx, send_idx, R.n_send * sizeof(long long), cudaMemcpyHostToDevice));
  }
  if (R.n_recv > 0) {
    CUCK(cudaMalloc(&R.d_recv_idx, R.n_recv * sizeof(long long)));
    CUCK(cudaMemcpy(R.d_recv_idx, recv_idx, R.n_recv * sizeof(long long), cudaMemcpyHostToDevice));
  }
  if (loop_) loop_->row_send_off[which][rank_] = R.send_off;
  R.ready = true;
  return true;
}

bool Comm::exchange_rows(double* field, int which, cudaStream_t st) {
  if (nranks_ <= 1) return true;
  RowPlan& R = rows_[which];
  if (!R.ready) {
    err_ = "face-row plan not set";
    return false;
  }
  const size_t need = (size_t)std::max(R.n_send, R.n_recv);
  auto grid_for = [](long long n) { return (int)std::min<long long>((n + 255) / 256, 4096); };
  if (loop_) {
    LoopGroup* G = loop_;
    for (int q = 0; q < nranks_; ++q)
      if (q != rank_) CUCK(cudaStreamWaitEvent(st, G->ev_copied[q], 0));
    if (!ensure_cap(need)) return false;
    if (R.n_send > 0) {
      k_pack_idx<<<grid_for(R.n_send), 256, 0, st>>>(field, R.d_send_idx, R.n_send, sendbuf_);
      CUCK(cudaGetLastError());
    }
    CUCK(cudaEventRecord(G->ev_pack[rank_], st));
    G->sendbuf[rank_] = sendbuf_;
    G->barrier();
    for (int q = 0; q < nranks_; ++q) {
      const long long cnt = R.recv_off[q + 1] - R.recv_off[q];
      if (q == rank_ || cnt == 0) continue;
      CUCK(cudaStreamWaitEvent(st, G->ev_pack[q], 0));
      CUCK(cudaMemcpyAsync(recvbuf_ + R.recv_off[q],
                           G->sendbuf[q] + G->row_send_off[which][q][rank_],
                           (size_t)cnt * sizeof(double), cudaMemcpyDeviceToDevice, st));
    }
    CUCK(cudaEventRecord(G->ev_copied[rank_], st));
    G->barrier();
    if (R.n_recv > 0) {
      k_unpack_idx<<<grid_for(R.n_recv), 256, 0, st>>>(field, R.d_recv_idx, R.n_recv, recvbuf_);
      CUCK(cudaGetLastError());
    }
    return true;
  }
  if (!ensure_cap(need)) return false;
  if (R.n_send > 0) {
    k_pack_idx<<<grid_for(R.n_send), 256, 0, st>>>(field, R.d_send_idx, R.n_send, sendbuf_);
    CUCK(cudaGetLastError());
  }
  ncclComm_t c = (ncclComm_t)comm_;
  NCCK(ncclGroupStart());
  for (int p = 0; p < nranks_; ++p) {
    if (p == rank_) continue;
    const long long ns = R.send_off[p + 1] - R.send_off[p], nr = R.recv_off[p + 1] - R.recv_off[p];
    if (ns > 0) NCCK(ncclSend(sendbuf_ + R.send_off[p], (size_t)ns, ncclDouble, p, c, st));
    if (nr > 0) NCCK(ncclRecv(recvbuf_ + R.recv_off[p], (size_t)nr, ncclDouble, p, c, st));
  }
  NCCK(ncclGroupEnd());
  if (R.n_recv > 0) {
    k_unpack_idx<<<grid_for(R.n_recv), 256, 0, st>>>(field, R.d_recv_idx, R.n_recv, recvbuf_);
    CUCK(cudaGetLastError());
  }
  return true;
}

bool Comm::allreduce_sum(double* dev, int n, cudaStream_t st) {
  if (nranks_ <= 1) return true;
  if (loop_) return loop_reduce(dev, n, st, 0);
  NCCK(ncclAllReduce(dev, dev, n, ncclDouble, ncclSum, (ncclComm_t)comm_, st));
  return true;
}

bool Comm::allreduce_max(double* dev, int n, cudaStream_t st) {
  if (nranks_ <= 1) return true;
  if (loop_) return loop_reduce(dev, n, st, 1);
  NCCK(ncclAllReduce(dev, dev, n, ncclDouble, ncclMax, (ncclComm_t)comm_, st));
  return true;
}

bool Comm::allreduce_minloc(double loc[4], cudaStream_t st) {
  if (nranks_ <= 1) return true;
  if (loop_) {
    LoopGroup* G = loop_;
    auto& mine = G->slots[rank_];
    if (mine.size() < 4) mine.resize(4);
    std::copy(loc, loc + 4, mine.begin());
    G->barrier();
    double v[2] = {INFINITY, INFINITY}, idx[2] = {INFINITY, INFINITY};
    for (int q = 0; q < G->n; ++q)
      for (int k = 0; k < 2; ++k) v[k] = std::min(v[k], G->slots[q][2 * k]);
    for (int q = 0; q < G->n; ++q)
      for (int k = 0; k < 2; ++k)
        if (G->slots[q][2 * k] == v[k]) idx[k] = std::min(idx[k], G->slots[q][2 * k + 1]);
    G->barrier();
    loc[0] = v[0];
    loc[1] = idx[0];
    loc[2] = v[1];
    loc[3] = idx[1];
    return true;
  }
  ncclComm_t c = (ncclComm_t)comm_;
  double v[2] = {loc[0], loc[2]};
  CUCK(cudaMemcpyAsync(scratch_, v, 2 * sizeof(double), cudaMemcpyHostToDevice, st));
  NCCK(ncclAllReduce(scratch_, scratch_, 2, ncclDouble, ncclMin, c, st));
  CUCK(cudaMemcpyAsync(v, scratch_, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
  CUCK(cudaStreamSynchronize(st));
  double idx[2] = {loc[0] == v[0] ? loc[1] : INFINITY, loc[2] == v[1] ? loc[3] : INFINITY};
  CUCK(cudaMemcpyAsync(scratch_, idx, 2 * sizeof(double), cudaMemcpyHostToDevice, st));
  NCCK(ncclAllReduce(scratch_, scratch_, 2, ncclDouble, ncclMin, c, st));
  CUCK(cudaMemcpyAsync(idx, scratch_, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
  CUCK(cudaStreamSynchronize(st));
  loc[0] = v[0];
  loc[1] = idx[0];
  loc[2] = v[1];
  loc[3] = idx[1];
  return true;
}

void Comm::shutdown() {
  if (comm_) ncclCommDestroy((ncclComm_t)comm_);
  comm_ = nullptr;
  loop_ = nullptr;
  if (d_send_elems_) cudaFree(d_send_elems_);
  if (sendbuf_) cudaFree(sendbuf_);
  if (recvbuf_) cudaFree(recvbuf_);
  if (scratch_) cudaFree(scratch_);
  for (auto& R : rows_) {
    if (R.d_send_idx) cudaFree(R.d_send_idx);
    if (R.d_recv_idx) cudaFree(R.d_recv_idx);
    R = RowPlan{};
  }
  d_send_elems_ = nullptr;
  sendbuf_ = recvbuf_ = scratch_ = nullptr;
  buf_cap_ = 0;
  nranks_ = 1;
}

}  // namespace dg
