// NcclComm and ThreadComm (see comm.hpp).
#include "comm.hpp"

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "device.hpp"
#include "kernels.h"

namespace pdlp_host {

// ------------------------------------------------------------------ NCCL ---
namespace {

struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*reduce_scatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t,
                                 ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;

  NcclApi() {
    // The soname torch's bundled NCCL also carries: if torch loaded it first
    // the same library is reused.
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (h == nullptr) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
    if (h == nullptr) {
      const char* e = dlerror();
      why = std::string("libnccl not loadable: ") + (e ? e : "?");
      return;
    }
    bool all = true;
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      if (fn == nullptr) all = false;
    };
    sym(get_unique_id, "ncclGetUniqueId");
    sym(comm_init_rank, "ncclCommInitRank");
    sym(comm_destroy, "ncclCommDestroy");
    sym(all_gather, "ncclAllGather");
    sym(reduce_scatter, "ncclReduceScatter");
    sym(all_reduce, "ncclAllReduce");
    sym(error_string, "ncclGetErrorString");
    ok = all;
    if (!all) why = "libnccl is missing an entry point";
  }
};

NcclApi& nccl() {
  static NcclApi api;
  return api;
}

void check_nccl(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    throw CudaError(std::string(what) + ": " + nccl().error_string(r));
  }
}

class NcclComm final : public Comm {
 public:
  NcclComm(const unsigned char id[128], int rank, int world, int device) : rank_(rank), world_(world) {
    NcclApi& api = nccl();
    if (!api.ok) throw CudaError(api.why);
    PDLP_CK(cudaSetDevice(device));
    ncclUniqueId uid;
    static_assert(sizeof(uid.internal) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(uid.internal, id, 128);
    check_nccl(api.comm_init_rank(&comm_, world, uid, rank), "ncclCommInitRank");
  }

  int rank() const override { return rank_; }
  int world() const override { return world_; }
  void allgather(double* buf, size_t count, cudaStream_t s) override {
    if (count == 0) return;
    check_nccl(nccl().all_gather(buf + count * rank_, buf, count, ncclDouble, comm_, s),
               "ncclAllGather");
  }
  void reduce_scatter(const double* send, double* recv, size_t count, cudaStream_t s) override {
    if (count == 0) return;
    check_nccl(nccl().reduce_scatter(send, recv, count, ncclDouble, ncclSum, comm_, s),
               "ncclReduceScatter");
  }
  void allreduce(double* buf, size_t count, bool use_max, cudaStream_t s) override {
    if (count == 0) return;
    check_nccl(nccl().all_reduce(buf, buf, count, ncclDouble, use_max ? ncclMax : ncclSum, comm_, s),
               "ncclAllReduce");
  }
  void barrier(cudaStream_t s) override {
    if (token_ == nullptr) PDLP_CK(cudaMalloc(&token_, sizeof(double)));
    check_nccl(nccl().all_reduce(token_, token_, 1, ncclDouble, ncclSum, comm_, s), "ncclAllReduce");
  }
  std::vector<double*> peer_pointers(double* mine, cudaStream_t s) override {
    // Exchange CUDA IPC handles (64 bytes per rank) with one all-gather.  A
    // local failure still takes part in the exchange (all-zero handle) and
    // returns an empty vector, so no peer is left waiting in a collective.
    const size_t hb = sizeof(cudaIpcMemHandle_t);
    std::vector<char> all(hb * world_, 0);
    bool ok = cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t*>(all.data() + hb * rank_),
                                  mine) == cudaSuccess;
    cudaGetLastError();
    char* dev = nullptr;
    PDLP_CK(cudaMalloc(&dev, hb * world_));
    PDLP_CK(cudaMemcpyAsync(dev, all.data(), hb * world_, cudaMemcpyHostToDevice, s));
    check_nccl(nccl().all_gather(dev + hb * rank_, dev, hb, ncclChar, comm_, s), "ncclAllGather");
    PDLP_CK(cudaMemcpyAsync(all.data(), dev, hb * world_, cudaMemcpyDeviceToHost, s));
    PDLP_CK(cudaStreamSynchronize(s));
    cudaFree(dev);
    std::vector<double*> out(static_cast<size_t>(world_), nullptr);
    for (int r = 0; r < world_ && ok; ++r) {
      if (r == rank_) {
        out[r] = mine;
        continue;
      }
      cudaIpcMemHandle_t peer;
      std::memcpy(&peer, all.data() + hb * r, hb);
      void* p = nullptr;
      if (cudaIpcOpenMemHandle(&p, peer, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        ok = false;
        break;
      }
      opened_.push_back(p);
      out[r] = static_cast<double*>(p);
    }
    if (!ok) {
      for (void* p : opened_) cudaIpcCloseMemHandle(p);
      opened_.clear();
      out.clear();
    }
    return out;
  }
  double* alloc_peer_buffer(size_t count) override {
    double* p = nullptr;
    PDLP_CK(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(double)));
    return p;
  }
  void free_peer_buffer(double* p) override { cudaFree(p); }
  ~NcclComm() override {
    for (void* p : opened_) cudaIpcCloseMemHandle(p);
    if (token_ != nullptr) cudaFree(token_);
    if (comm_ != nullptr) nccl().comm_destroy(comm_);
  }

 private:
  int rank_, world_;
  ncclComm_t comm_ = nullptr;
  double* token_ = nullptr;
  std::vector<void*> opened_;
};

}  // namespace

std::unique_ptr<Comm> make_nccl_comm(const unsigned char id[128], int rank, int world, int device) {
  return std::make_unique<NcclComm>(id, rank, world, device);
}

bool nccl_unique_id(unsigned char id[128], const char** why) {
  NcclApi& api = nccl();
  if (!api.ok) {
    if (why) *why = api.why.c_str();
    return false;
  }
  ncclUniqueId uid;
  const ncclResult_t r = api.get_unique_id(&uid);
  if (r != ncclSuccess) {
    if (why) *why = api.error_string(r);
    return false;
  }
  std::memcpy(id, uid.internal, 128);
  return true;
}

// ----------------------------------------------------------- ThreadComm ---
struct ThreadHub {
  int world = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t phase = 0;
  bool aborted = false;
  std::vector<const double*> ptr;

  void barrier() {
    std::unique_lock<std::mutex> g(mu);
    if (aborted) throw CudaError("another rank of the group failed");
    const uint64_t my = phase;
    if (++arrived == world) {
      arrived = 0;
      ++phase;
      cv.notify_all();
      return;
    }
    cv.wait(g, [&] { return phase != my || aborted; });
    if (aborted) throw CudaError("another rank of the group failed");
  }
};

std::shared_ptr<ThreadHub> make_thread_hub(int world) {
  auto h = std::make_shared<ThreadHub>();
  h->world = world;
  h->ptr.assign(static_cast<size_t>(world), nullptr);
  return h;
}

void abort_thread_hub(ThreadHub& hub) {
  std::lock_guard<std::mutex> g(hub.mu);
  hub.aborted = true;
  hub.cv.notify_all();
}

namespace {

class ThreadComm final : public Comm {
 public:
  ThreadComm(std::shared_ptr<ThreadHub> hub, int rank) : hub_(std::move(hub)), rank_(rank) {}
  int rank() const override { return rank_; }
  int world() const override { return hub_->world; }

  // Publish a pointer once this rank's stream has produced it.
  void publish(const double* p, cudaStream_t s) {
    PDLP_CK(cudaStreamSynchronize(s));
    hub_->ptr[static_cast<size_t>(rank_)] = p;
    hub_->barrier();
  }
  // Leave once every rank has finished reading the published buffers.
  void release(cudaStream_t s) {
    PDLP_CK(cudaStreamSynchronize(s));
    hub_->barrier();
  }

  void allgather(double* buf, size_t count, cudaStream_t s) override {
    publish(buf, s);
    for (int r = 0; r < world(); ++r) {
      if (r == rank_ || count == 0) continue;
      PDLP_CK(cudaMemcpyAsync(buf + count * r, hub_->ptr[r] + count * r, count * sizeof(double),
                              cudaMemcpyDeviceToDevice, s));
    }
    release(s);
  }
  void reduce_scatter(const double* send, double* recv, size_t count, cudaStream_t s) override {
    publish(send, s);
    if (count > 0) {
      PDLP_CK(cudaMemcpyAsync(recv, hub_->ptr[0] + count * rank_, count * sizeof(double),
                              cudaMemcpyDeviceToDevice, s));
      for (int r = 1; r < world(); ++r) {
        PDLP_LAUNCH(pdlpk_accumulate(recv, hub_->ptr[r] + count * rank_, static_cast<int64_t>(count),
                                     0, s));
      }
    }
    release(s);
  }
  void barrier(cudaStream_t s) override {
    publish(nullptr, s);
    release(s);
  }
  std::vector<double*> peer_pointers(double* mine, cudaStream_t s) override {
    publish(mine, s);
    std::vector<double*> out(static_cast<size_t>(world()));
    for (int r = 0; r < world(); ++r) out[r] = const_cast<double*>(hub_->ptr[r]);
    release(s);
    return out;
  }
  double* alloc_peer_buffer(size_t count) override {
    double* p = nullptr;
    PDLP_CK(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(double)));
    return p;
  }
  void free_peer_buffer(double* p) override { cudaFree(p); }
  void allreduce(double* buf, size_t count, bool use_max, cudaStream_t s) override {
    DevBuf<double> tmp(count);
    publish(buf, s);
    if (count > 0) {
      PDLP_CK(cudaMemcpyAsync(tmp.get(), hub_->ptr[0], count * sizeof(double),
                              cudaMemcpyDeviceToDevice, s));
      for (int r = 1; r < world(); ++r) {
        PDLP_LAUNCH(pdlpk_accumulate(tmp.get(), hub_->ptr[r], static_cast<int64_t>(count),
                                     use_max ? 1 : 0, s));
      }
    }
    release(s);
    if (count > 0) {
      PDLP_CK(cudaMemcpyAsync(buf, tmp.get(), count * sizeof(double), cudaMemcpyDeviceToDevice, s));
    }
  }

 private:
  std::shared_ptr<ThreadHub> hub_;
  int rank_;
};

}  // namespace

std::unique_ptr<Comm> make_thread_comm(std::shared_ptr<ThreadHub> hub, int rank) {
  return std::make_unique<ThreadComm>(std::move(hub), rank);
}

}  // namespace pdlp_host
