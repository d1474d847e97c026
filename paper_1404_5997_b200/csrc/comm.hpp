// Worker-to-worker transport for the step's exchange points
// (exchange_activations / return_gradients / fc-internal gather+reduce /
// sync_conv_gradients, cluster.cpp:157-319, 534-584).
//
//   LogicalComm: all K workers live on this device in one process; each
//     collective is stream-ordered device copies / reduction kernels that sum
//     in ascending worker order (the reference's order). Used for parity on
//     one GPU and for the routing tests.
//   NcclComm: one worker per process (torchrun, one GPU each); collectives
//     are NCCL over NVLink / NVSwitch.
//
// Every call takes one buffer per LOCAL worker (K for logical, 1 for NCCL).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <memory>
#include <vector>

namespace hp {

class Comm {
 public:
  virtual ~Comm() = default;
  virtual int world() const = 0;   // K
  virtual int nlocal() const = 0;  // local workers
  virtual int first() const = 0;   // global id of local worker 0

  // bufs[w]: K chunks of `bytes`; chunk g is valid in worker g's buffer on entry,
  // every chunk is valid everywhere on exit (ncclAllGather in place).
  virtual void allgather_inplace(const std::vector<void*>& bufs, size_t bytes, cudaStream_t s) = 0;
  // send[w] (bytes) -> recv[w] chunk (global id of w).
  virtual void allgather(const std::vector<const void*>& send, const std::vector<void*>& recv,
                         size_t bytes, cudaStream_t s) = 0;
  // bufs[w]: root's buffer is the source (ncclBroadcast in place).
  virtual void broadcast(const std::vector<void*>& bufs, size_t bytes, int root, cudaStream_t s) = 0;
  // send[w]: K chunks of `count` fp32 -> recv[w] = alpha * sum over workers of chunk (global id
  // of w), written as out_type (0 fp32, 1 bf16).
  virtual void reduce_scatter(const std::vector<const float*>& send, const std::vector<void*>& recv,
                              size_t count, int out_type, float alpha, cudaStream_t s) = 0;
  // recv (valid on the root only; nullptr elsewhere) = alpha * sum of send[w].
  virtual void reduce(const std::vector<const float*>& send, void* recv_root, size_t count, int root,
                      int out_type, float alpha, cudaStream_t s) = 0;
  // bufs[w] = sum over workers (fp32 / fp64).
  virtual void allreduce_f32(const std::vector<float*>& bufs, size_t count, cudaStream_t s) = 0;
  virtual void allreduce_f64(const std::vector<double*>& bufs, size_t count, cudaStream_t s) = 0;
  // Scratch reservation for fp32 staging (NCCL reduce -> cast).
  virtual void reserve(size_t bytes) = 0;
  // A transport over the same workers for use on another stream (NCCL: a new
  // communicator from ncclCommSplit, so concurrent streams never share one).
  virtual std::unique_ptr<Comm> split() = 0;
  // Throws HP_ERR_NCCL if the transport saw an asynchronous failure (a peer
  // died, a network error); the communicator is aborted first so pending
  // collectives return instead of hanging.
  virtual void check_async() {}
};

std::unique_ptr<Comm> make_logical_comm(int K);
std::unique_ptr<Comm> make_nccl_comm(int K, int rank, const unsigned char id[128]);
void nccl_unique_id(unsigned char out[128]);

}  // namespace hp
