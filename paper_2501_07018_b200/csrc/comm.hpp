// Collectives of the row-sharded solve.
//
// One process (or host thread) per rank; every rank runs the same host
// program (SPMD) and calls the collectives in the same order.  Buffers are
// device memory; calls are ordered on the caller's stream.
//
//   NcclComm    one GPU per rank over NCCL (NVLink / NVSwitch).  libnccl is
//               opened at run time, so single-GPU solves never depend on it.
//   ThreadComm  `world` ranks as host threads of one process sharing one
//               GPU, each with its own stream.  A collective is a host
//               barrier plus device-to-device copies and rank-ordered adds;
//               no kernel ever waits on another rank's kernel, so it is safe
//               on a single GPU.  It exists to run the sharded code path with
//               world > 1 where only one GPU is available (tests).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <memory>
#include <vector>

namespace pdlp_host {

class Comm {
 public:
  virtual ~Comm() = default;
  virtual int rank() const = 0;
  virtual int world() const = 0;
  // In place: buf holds world blocks of `count` doubles; block rank() is this
  // rank's input, every block is filled on return (in stream order).
  virtual void allgather(double* buf, size_t count, cudaStream_t s) = 0;
  // send: world blocks of `count`; recv (count) = sum over ranks of block rank().
  virtual void reduce_scatter(const double* send, double* recv, size_t count, cudaStream_t s) = 0;
  // In place elementwise sum (or max) over ranks.
  virtual void allreduce(double* buf, size_t count, bool use_max, cudaStream_t s) = 0;
  // Stream-level barrier: work enqueued on every rank's stream before the
  // call is complete before work enqueued after it runs (no kernel spins).
  virtual void barrier(cudaStream_t s) = 0;
  // Every rank's address of a buffer each rank allocated with
  // alloc_peer_buffer (collective; index = rank).  NVLink P2P across
  // processes (CUDA IPC), plain pointers for ranks sharing a process.
  // Empty if this rank could not map its peers (the caller agrees on a
  // fallback with the other ranks).
  virtual std::vector<double*> peer_pointers(double* mine, cudaStream_t s) = 0;
  // Device memory that peers can map (not from the stream-ordered pool).
  virtual double* alloc_peer_buffer(size_t count) = 0;
  virtual void free_peer_buffer(double* p) = 0;
};

// NCCL communicator from a 128-byte ncclUniqueId created by rank 0 and
// shared out of band (torch.distributed in the Python launcher).
std::unique_ptr<Comm> make_nccl_comm(const unsigned char id[128], int rank, int world,
                                     int device);
// Writes a fresh ncclUniqueId; returns false (with a message) if libnccl is
// unavailable.
bool nccl_unique_id(unsigned char id[128], const char** why);

// Shared state of a ThreadComm group; create once, then one comm per thread.
struct ThreadHub;
std::shared_ptr<ThreadHub> make_thread_hub(int world);
std::unique_ptr<Comm> make_thread_comm(std::shared_ptr<ThreadHub> hub, int rank);
// Releases every thread blocked in a collective of the hub (error path).
void abort_thread_hub(ThreadHub& hub);

}  // namespace pdlp_host
