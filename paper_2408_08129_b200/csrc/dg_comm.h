// Multi-GPU plumbing of libdg: one process per GPU, NCCL over NVLink /
// NVSwitch.  Two collectives only:
//   * halo exchange of ghost ELEMENTS before every face-coupled operator
//     (grouped ncclSend/ncclRecv to each neighbour rank; ghosts are stored
//     after the owned elements, ordered by (owner rank, global id), so each
//     peer's ghosts form one contiguous block);
//   * allreduce of the Krylov / fixed-point / diagnostic scalars.
// With nranks == 1 every call is a no-op and NCCL is never initialised.
// A loopback backend (init_loopback) runs the same plans between contexts of
// one process -- the executable test of the multi-rank path on one GPU.
#pragma once
#include <cstdint>
#include <string>
#include <vector>
#include <cuda_runtime.h>

namespace dg {

struct LoopGroup;

class Comm {
 public:
  static bool unique_id(void* out128, std::string* err);
  bool init(const void* uid, int rank, int nranks, const int32_t* send_counts,
            const int32_t* send_elems, const int32_t* recv_counts, int n_el, int n_tot);
  // loopback backend: nranks contexts of ONE process (one host thread each,
  // same or different devices) forming group `group`; the exchange is one
  // cudaMemcpyAsync per peer ordered by CUDA events and host barriers, the
  // allreduces sum the ranks' values on the host in rank order.  No kernel
  // ever waits on another rank's kernel.  Every rank must call it.
  bool init_loopback(int group, int rank, int nranks, const int32_t* send_counts,
                     const int32_t* send_elems, const int32_t* recv_counts, int n_el, int n_tot);
  bool active() const { return nranks_ > 1; }
  bool exchange(double* field, int ncomp, int np, cudaStream_t st, long long estride = -1);
  bool allreduce_sum(double* dev, int n, cudaStream_t st);
  bool allreduce_max(double* dev, int n, cudaStream_t st);
  bool allreduce_minloc(double loc[4], cudaStream_t st);  // (v0, i0, v1, i1) global min
  long long global_index(long long local) const { return offset_ + local; }
  const std::string& error() const { return err_; }
  void shutdown();

 private:
  void* comm_ = nullptr;  // ncclComm_t
  LoopGroup* loop_ = nullptr;
  bool init_plan(int rank, int nranks, const int32_t* send_counts, const int32_t* send_elems,
                 const int32_t* recv_counts, int n_el, int n_tot);
  bool ensure_bufs(size_t per);
  bool loop_reduce(double* dev, int n, cudaStream_t st, int op);
  int rank_ = 0, nranks_ = 1, n_el_ = 0, n_tot_ = 0;
  long long offset_ = 0;
  std::vector<int> send_counts_, recv_counts_, send_off_, recv_off_;
  int* d_send_elems_ = nullptr;
  int n_send_ = 0;
  double* sendbuf_ = nullptr;
  double* recvbuf_ = nullptr;
  size_t buf_cap_ = 0;
  double* scratch_ = nullptr;
  std::string err_;
};

}  // namespace dg
