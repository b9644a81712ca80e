// NCCL halo exchange and allreduces of libdg (see dg_comm.h).
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>

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
  const size_t need = std::max((size_t)n_send_, (size_t)(n_tot_ - n_el_)) * per;
  if (need > buf_cap_) {
    if (sendbuf_) cudaFree(sendbuf_);
    if (recvbuf_) cudaFree(recvbuf_);
    CUCK(cudaMalloc(&sendbuf_, need * sizeof(double)));
    CUCK(cudaMalloc(&recvbuf_, need * sizeof(double)));
    buf_cap_ = need;
  }
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

bool Comm::allreduce_sum(double* dev, int n, cudaStream_t st) {
  if (nranks_ <= 1) return true;
  NCCK(ncclAllReduce(dev, dev, n, ncclDouble, ncclSum, (ncclComm_t)comm_, st));
  return true;
}

bool Comm::allreduce_max(double* dev, int n, cudaStream_t st) {
  if (nranks_ <= 1) return true;
  NCCK(ncclAllReduce(dev, dev, n, ncclDouble, ncclMax, (ncclComm_t)comm_, st));
  return true;
}

bool Comm::allreduce_minloc(double loc[4], cudaStream_t st) {
  if (nranks_ <= 1) return true;
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
  if (d_send_elems_) cudaFree(d_send_elems_);
  if (sendbuf_) cudaFree(sendbuf_);
  if (recvbuf_) cudaFree(recvbuf_);
  if (scratch_) cudaFree(scratch_);
  d_send_elems_ = nullptr;
  sendbuf_ = recvbuf_ = scratch_ = nullptr;
  buf_cap_ = 0;
  nranks_ = 1;
}

}  // namespace dg
