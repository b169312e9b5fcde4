#include "dist.hpp"

#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

namespace gb {

namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA error ") + cudaGetErrorString(e) + " in " + what);
}

// ------------------------------------------------------------------ NCCL
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*errorString)(ncclResult_t) = nullptr;

  static NcclApi& get() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
      for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
        api.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
        if (api.h) break;
      }
      if (!api.h) return;
      api.getUniqueId = reinterpret_cast<decltype(api.getUniqueId)>(dlsym(api.h, "ncclGetUniqueId"));
      api.commInitRank = reinterpret_cast<decltype(api.commInitRank)>(dlsym(api.h, "ncclCommInitRank"));
      api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(dlsym(api.h, "ncclCommDestroy"));
      api.allReduce = reinterpret_cast<decltype(api.allReduce)>(dlsym(api.h, "ncclAllReduce"));
      api.broadcast = reinterpret_cast<decltype(api.broadcast)>(dlsym(api.h, "ncclBroadcast"));
      api.errorString = reinterpret_cast<decltype(api.errorString)>(dlsym(api.h, "ncclGetErrorString"));
    });
    if (!api.h || !api.allReduce || !api.commInitRank)
      throw std::runtime_error("NCCL (libnccl.so.2) not loadable: required for multi-GPU sharding");
    return api;
  }
  void check(ncclResult_t r, const char* what) const {
    if (r != ncclSuccess)
      throw std::runtime_error(std::string("NCCL error in ") + what + ": " + (errorString ? errorString(r) : "?"));
  }
};

class NcclReducer final : public Reducer {
 public:
  NcclReducer(int world, int rank, const void* id) : world_(world), rank_(rank) {
    NcclApi& api = NcclApi::get();
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    api.check(api.commInitRank(&comm_, world, uid, rank), "ncclCommInitRank");
  }
  ~NcclReducer() override {
    if (comm_) NcclApi::get().commDestroy(comm_);
  }
  int world() const override { return world_; }
  int rank() const override { return rank_; }
  bool capturable() const override { return true; }
  void allreduce(void* buf, size_t count, int eb, bool max, cudaStream_t s) override {
    NcclApi& api = NcclApi::get();
    api.check(api.allReduce(buf, buf, count, eb == 8 ? ncclFloat64 : ncclFloat32, max ? ncclMax : ncclSum, comm_, s),
              "ncclAllReduce");
  }
  void broadcast(void* buf, size_t bytes, int root, cudaStream_t s) override {
    NcclApi& api = NcclApi::get();
    api.check(api.broadcast(buf, buf, bytes, ncclUint8, root, comm_, s), "ncclBroadcast");
  }

 private:
  int world_, rank_;
  ncclComm_t comm_ = nullptr;
};

// -------------------------------------------------------------- loopback
constexpr int kMaxLoop = 16;
struct PtrList {
  const void* p[kMaxLoop];
};

template <typename T>
__global__ void k_loop_reduce(PtrList in, int world, size_t n, bool max, T* out) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    T acc = static_cast<const T*>(in.p[0])[i];
    for (int r = 1; r < world; ++r) {
      const T v = static_cast<const T*>(in.p[r])[i];
      acc = max ? (v > acc ? v : acc) : acc + v;
    }
    out[i] = acc;
  }
}

struct LoopGroup {
  int world = 0;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  void* bufs[kMaxLoop] = {};
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
  cudaStream_t stream = nullptr;
  ~LoopGroup() {
    if (scratch) cudaFree(scratch);
    if (stream) cudaStreamDestroy(stream);
  }
};

std::mutex g_loop_mu;
std::map<uint64_t, std::weak_ptr<LoopGroup>> g_loop_groups;

class LoopbackReducer final : public Reducer {
 public:
  LoopbackReducer(int world, int rank, uint64_t key) : world_(world), rank_(rank) {
    if (world > kMaxLoop) throw std::invalid_argument("loopback group larger than 16");
    std::lock_guard<std::mutex> lk(g_loop_mu);
    auto& w = g_loop_groups[key];
    group_ = w.lock();
    if (!group_) {
      group_ = std::make_shared<LoopGroup>();
      group_->world = world;
      w = group_;
    }
    if (group_->world != world) throw std::invalid_argument("loopback group size mismatch");
  }
  int world() const override { return world_; }
  int rank() const override { return rank_; }
  bool capturable() const override { return false; }

  // host rendezvous; the last arriving rank runs `work` for everybody
  template <typename F>
  void rendezvous(void* buf, F&& work) {
    LoopGroup& g = *group_;
    std::unique_lock<std::mutex> lk(g.m);
    g.bufs[rank_] = buf;
    const uint64_t my_gen = g.gen;
    if (++g.arrived == world_) {
      work(g);
      g.arrived = 0;
      ++g.gen;
      g.cv.notify_all();
    } else {
      g.cv.wait(lk, [&] { return g.gen != my_gen; });
    }
  }

  void allreduce(void* buf, size_t count, int eb, bool max, cudaStream_t s) override {
    ck(cudaStreamSynchronize(s), "loopback allreduce");
    rendezvous(buf, [&](LoopGroup& g) {
      if (!g.stream) ck(cudaStreamCreateWithFlags(&g.stream, cudaStreamNonBlocking), "loopback stream");
      const size_t bytes = count * static_cast<size_t>(eb);
      if (g.scratch_bytes < bytes) {
        if (g.scratch) cudaFree(g.scratch);
        ck(cudaMalloc(&g.scratch, bytes), "loopback scratch");
        g.scratch_bytes = bytes;
      }
      PtrList pl{};
      for (int r = 0; r < world_; ++r) pl.p[r] = g.bufs[r];
      const unsigned grid = static_cast<unsigned>(std::min<size_t>((count + 255) / 256, 1024));
      if (eb == 8)
        k_loop_reduce<double><<<grid ? grid : 1, 256, 0, g.stream>>>(pl, world_, count, max, static_cast<double*>(g.scratch));
      else
        k_loop_reduce<float><<<grid ? grid : 1, 256, 0, g.stream>>>(pl, world_, count, max, static_cast<float*>(g.scratch));
      ck(cudaGetLastError(), "loopback reduce");
      for (int r = 0; r < world_; ++r)
        ck(cudaMemcpyAsync(g.bufs[r], g.scratch, bytes, cudaMemcpyDeviceToDevice, g.stream), "loopback copy");
      ck(cudaStreamSynchronize(g.stream), "loopback sync");
    });
  }

  void broadcast(void* buf, size_t bytes, int root, cudaStream_t s) override {
    ck(cudaStreamSynchronize(s), "loopback broadcast");
    rendezvous(buf, [&](LoopGroup& g) {
      if (!g.stream) ck(cudaStreamCreateWithFlags(&g.stream, cudaStreamNonBlocking), "loopback stream");
      for (int r = 0; r < world_; ++r)
        if (r != root) ck(cudaMemcpyAsync(g.bufs[r], g.bufs[root], bytes, cudaMemcpyDeviceToDevice, g.stream), "copy");
      ck(cudaStreamSynchronize(g.stream), "loopback sync");
    });
  }

 private:
  int world_, rank_;
  std::shared_ptr<LoopGroup> group_;
};

}  // namespace

std::unique_ptr<Reducer> make_reducer(int kind, int world, int rank, const void* id) {
  if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("invalid world/rank");
  if (kind == 0) return std::make_unique<NcclReducer>(world, rank, id);
  if (kind == 1) {
    uint64_t key = 0;
    std::memcpy(&key, id, sizeof(key));
    return std::make_unique<LoopbackReducer>(world, rank, key);
  }
  throw std::invalid_argument("unknown reducer kind");
}

void nccl_unique_id(void* out128) {
  NcclApi& api = NcclApi::get();
  ncclUniqueId uid;
  api.check(api.getUniqueId(&uid), "ncclGetUniqueId");
  std::memcpy(out128, &uid, sizeof(uid));
}

}  // namespace gb
