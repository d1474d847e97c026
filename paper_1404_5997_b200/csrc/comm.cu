// Logical and NCCL transports. See comm.hpp.
#include <nccl.h>

#include <cstring>
#include <string>

#include "comm.hpp"
#include "errors.hpp"
#include "kernels.cuh"

namespace hp {

namespace {

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    throw Error(HP_ERR_NCCL, std::string(what) + ": " + ncclGetErrorString(r));
  }
}
#define HP_NCCL(x) nccl_check((x), #x)

void finish_f32(const float* src, void* dst, size_t count, int out_type, float alpha,
                cudaStream_t s) {
  PtrList l{};
  l.p[0] = src;
  if (out_type == 1) {
    launch_sum_k<bf16>(l, 1, static_cast<bf16*>(dst), static_cast<long long>(count), alpha, s);
  } else {
    launch_sum_k<float>(l, 1, static_cast<float*>(dst), static_cast<long long>(count), alpha, s);
  }
}

class LogicalComm final : public Comm {
 public:
  explicit LogicalComm(int K) : K_(K) {
    if (K > kMaxLocal) config_error("cluster.workers: logical transport supports at most 16 workers");
  }
  int world() const override { return K_; }
  int nlocal() const override { return K_; }
  int first() const override { return 0; }

  void allgather_inplace(const std::vector<void*>& bufs, size_t bytes, cudaStream_t s) override {
    for (int d = 0; d < K_; ++d)
      for (int g = 0; g < K_; ++g) {
        if (g == d) continue;
        HP_CUDA(cudaMemcpyAsync(static_cast<char*>(bufs[d]) + g * bytes,
                                static_cast<const char*>(bufs[g]) + g * bytes, bytes,
                                cudaMemcpyDeviceToDevice, s));
      }
  }
  void allgather(const std::vector<const void*>& send, const std::vector<void*>& recv, size_t bytes,
                 cudaStream_t s) override {
    for (int d = 0; d < K_; ++d)
      for (int g = 0; g < K_; ++g)
        HP_CUDA(cudaMemcpyAsync(static_cast<char*>(recv[d]) + g * bytes, send[g], bytes,
                                cudaMemcpyDeviceToDevice, s));
  }
  void broadcast(const std::vector<void*>& bufs, size_t bytes, int root, cudaStream_t s) override {
    for (int d = 0; d < K_; ++d)
      if (d != root)
        HP_CUDA(cudaMemcpyAsync(bufs[d], bufs[root], bytes, cudaMemcpyDeviceToDevice, s));
  }
  void reduce_scatter(const std::vector<const float*>& send, const std::vector<void*>& recv,
                      size_t count, int out_type, float alpha, cudaStream_t s) override {
    for (int r = 0; r < K_; ++r) {
      PtrList l{};
      for (int w = 0; w < K_; ++w) l.p[w] = send[w] + r * count;
      if (out_type == 1)
        launch_sum_k<bf16>(l, K_, static_cast<bf16*>(recv[r]), static_cast<long long>(count), alpha, s);
      else
        launch_sum_k<float>(l, K_, static_cast<float*>(recv[r]), static_cast<long long>(count), alpha, s);
    }
  }
  void reduce(const std::vector<const float*>& send, void* recv_root, size_t count, int root,
              int out_type, float alpha, cudaStream_t s) override {
    (void)root;
    PtrList l{};
    for (int w = 0; w < K_; ++w) l.p[w] = send[w];
    if (out_type == 1)
      launch_sum_k<bf16>(l, K_, static_cast<bf16*>(recv_root), static_cast<long long>(count), alpha, s);
    else
      launch_sum_k<float>(l, K_, static_cast<float*>(recv_root), static_cast<long long>(count), alpha, s);
  }
  void allreduce_f32(const std::vector<float*>& bufs, size_t count, cudaStream_t s) override {
    MutPtrList l{};
    for (int w = 0; w < K_; ++w) l.p[w] = bufs[w];
    launch_allreduce_k(l, K_, static_cast<long long>(count), s);
  }
  void allreduce_f64(const std::vector<double*>&, size_t, cudaStream_t) override {
    usage_error("allreduce_f64: not used with the logical transport");
  }
  void reserve(size_t) override {}
  std::unique_ptr<Comm> split() override { return std::make_unique<LogicalComm>(K_); }

 private:
  int K_;
};

class NcclComm final : public Comm {
 public:
  NcclComm(int K, int rank, const unsigned char id[128]) : K_(K), rank_(rank) {
    ncclUniqueId uid;
    static_assert(sizeof(uid.internal) == 128, "ncclUniqueId size");
    std::memcpy(uid.internal, id, 128);
    HP_NCCL(ncclCommInitRank(&comm_, K, uid, rank));
  }
  NcclComm(int K, int rank, ncclComm_t c) : K_(K), rank_(rank), comm_(c) {}
  ~NcclComm() override {
    if (comm_) ncclCommDestroy(comm_);
    if (scratch_) cudaFree(scratch_);
  }
  int world() const override { return K_; }
  int nlocal() const override { return 1; }
  int first() const override { return rank_; }

  void allgather_inplace(const std::vector<void*>& bufs, size_t bytes, cudaStream_t s) override {
    live();
    char* b = static_cast<char*>(bufs[0]);
    HP_NCCL(ncclAllGather(b + rank_ * bytes, b, bytes, ncclUint8, comm_, s));
  }
  void allgather(const std::vector<const void*>& send, const std::vector<void*>& recv, size_t bytes,
                 cudaStream_t s) override {
    live();
    HP_NCCL(ncclAllGather(send[0], recv[0], bytes, ncclUint8, comm_, s));
  }
  void broadcast(const std::vector<void*>& bufs, size_t bytes, int root, cudaStream_t s) override {
    live();
    HP_NCCL(ncclBroadcast(bufs[0], bufs[0], bytes, ncclUint8, root, comm_, s));
  }
  void reduce_scatter(const std::vector<const float*>& send, const std::vector<void*>& recv,
                      size_t count, int out_type, float alpha, cudaStream_t s) override {
    if (out_type == 0 && alpha == 1.f) {
      live();
    HP_NCCL(ncclReduceScatter(send[0], recv[0], count, ncclFloat32, ncclSum, comm_, s));
      return;
    }
    need(count * sizeof(float));
    live();
    HP_NCCL(ncclReduceScatter(send[0], scratch_, count, ncclFloat32, ncclSum, comm_, s));
    finish_f32(static_cast<const float*>(scratch_), recv[0], count, out_type, alpha, s);
  }
  void reduce(const std::vector<const float*>& send, void* recv_root, size_t count, int root,
              int out_type, float alpha, cudaStream_t s) override {
    const bool direct = out_type == 0 && alpha == 1.f;
    if (!direct) need(count * sizeof(float));
    void* dst = direct ? recv_root : scratch_;
    live();
    HP_NCCL(ncclReduce(send[0], dst, count, ncclFloat32, ncclSum, root, comm_, s));
    if (!direct && rank_ == root) finish_f32(static_cast<const float*>(scratch_), recv_root, count, out_type, alpha, s);
  }
  void allreduce_f32(const std::vector<float*>& bufs, size_t count, cudaStream_t s) override {
    live();
    HP_NCCL(ncclAllReduce(bufs[0], bufs[0], count, ncclFloat32, ncclSum, comm_, s));
  }
  void allreduce_f64(const std::vector<double*>& bufs, size_t count, cudaStream_t s) override {
    live();
    HP_NCCL(ncclAllReduce(bufs[0], bufs[0], count, ncclFloat64, ncclSum, comm_, s));
  }
  void reserve(size_t bytes) override { need(bytes); }
  std::unique_ptr<Comm> split() override {
    ncclComm_t c = nullptr;
    live();
    HP_NCCL(ncclCommSplit(comm_, 0, rank_, &c, nullptr));
    return std::make_unique<NcclComm>(K_, rank_, c);
  }
  void check_async() override {
    if (!comm_) return;
    ncclResult_t st = ncclSuccess;
    HP_NCCL(ncclCommGetAsyncError(comm_, &st));
    if (st == ncclSuccess || st == ncclInProgress) return;
    ncclCommAbort(comm_);
    comm_ = nullptr;
    throw Error(HP_ERR_NCCL, std::string("NCCL asynchronous error: ") + ncclGetErrorString(st) +
                                 " (communicator aborted)");
  }

 private:
  void live() const {
    if (!comm_) throw Error(HP_ERR_NCCL, "NCCL communicator was aborted after an asynchronous error");
  }
  void need(size_t bytes) {
    if (bytes <= scratch_bytes_) return;
    if (scratch_) {
      HP_CUDA(cudaDeviceSynchronize());
      HP_CUDA(cudaFree(scratch_));
    }
    HP_CUDA(cudaMalloc(&scratch_, bytes));
    scratch_bytes_ = bytes;
  }
  int K_, rank_;
  ncclComm_t comm_ = nullptr;
  void* scratch_ = nullptr;
  size_t scratch_bytes_ = 0;
};

}  // namespace

std::unique_ptr<Comm> make_logical_comm(int K) { return std::make_unique<LogicalComm>(K); }

std::unique_ptr<Comm> make_nccl_comm(int K, int rank, const unsigned char id[128]) {
  return std::make_unique<NcclComm>(K, rank, id);
}

void nccl_unique_id(unsigned char out[128]) {
  ncclUniqueId uid;
  HP_NCCL(ncclGetUniqueId(&uid));
  std::memcpy(out, uid.internal, 128);
}

}  // namespace hp
