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
  // face-row plans (SURVEY.md §8e "halo face-trace exchange"): instead of
  // whole ghost elements, only the values the owned elements' faces read --
  // the ghost's nodal face values of x, its psi row and (coarse parents) its
  // V trace slots on the shared face.  `which` names the field layout (0 x,
  // 1 psi, 2 trV); the index lists are offsets in doubles into the local
  // field, grouped by peer rank in the same (element, face) order on both
  // sides.  Every rank sets every plan (possibly empty) before its first use.
  static constexpr int N_ROW_PLANS = 3;
  bool set_rows(int which, const int64_t* send_counts, const int64_t* send_idx,
                const int64_t* recv_counts, const int64_t* recv_idx);
  bool has_rows() const { return rows_[0].ready && rows_[1].ready && rows_[2].ready; }
  bool exchange_rows(double* field, int which, cudaStream_t st);
  // doubles sent by this rank: per exchange_rows(which), and per whole-element
  // exchange of one value per node (accounting for tests / DESIGN.md)
  long long row_send_values(int which) const { return rows_[which].n_send; }
  long long elem_send_count() const { return n_send_; }
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
  bool ensure_cap(size_t need_values);
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
  struct RowPlan {
    bool ready = false;
    long long n_send = 0, n_recv = 0;
    std::vector<long long> send_off, recv_off;  // per-peer prefix sums
    long long* d_send_idx = nullptr;
    long long* d_recv_idx = nullptr;
  } rows_[N_ROW_PLANS];
  std::string err_;
};

}  // namespace dg
