#include "dist.hpp"

#include <dlfcn.h>
#include <fcntl.h>
#include <nccl.h>
#include <sched.h>
#include <sys/mman.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <thread>

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


// ------------------------------------------------------------ shared memory
// One process per rank on ONE host (and any GPUs, including all ranks on the
// same device): the collectives go through a POSIX shared-memory segment.
// allreduce: every rank copies its buffer into its own slot, a barrier, every
// rank sums the slots in rank order (identical bits on all ranks, like the
// loopback reducer), a second barrier before the slots are reused. Messages
// larger than a slot move in slot-sized pieces. Host-synchronous, so not
// capturable: the solver then launches each LM iteration eagerly.
struct ShmHeader {
  std::atomic<uint32_t> magic;
  std::atomic<uint32_t> arrived;
  std::atomic<uint32_t> gen;
  std::atomic<uint32_t> attached;
  uint32_t world;
  uint64_t slot_bytes;
};
static_assert(std::atomic<uint32_t>::is_always_lock_free, "process-shared atomics need lock-free uint32");
constexpr uint32_t kShmMagic = 0x67627368u;  // "gbsh"
constexpr uint64_t kShmSlot = uint64_t(8) << 20;

class ShmReducer final : public Reducer {
 public:
  ShmReducer(int world, int rank, uint64_t key) : world_(world), rank_(rank) {
    name_ = "/gb_shm_" + std::to_string(key);
    bytes_ = sizeof(ShmHeader) + 64 + static_cast<size_t>(world) * kShmSlot;
    const auto deadline = std::chrono::steady_clock::now() + std::chrono::seconds(120);
    int fd = -1;
    if (rank == 0) {
      shm_unlink(name_.c_str());  // a stale segment of a crashed run with the same key
      fd = shm_open(name_.c_str(), O_CREAT | O_EXCL | O_RDWR, 0600);
      if (fd < 0 || ftruncate(fd, static_cast<off_t>(bytes_)) != 0)
        throw std::runtime_error("shm reducer: cannot create " + name_);
    } else {
      while ((fd = shm_open(name_.c_str(), O_RDWR, 0600)) < 0) {
        if (std::chrono::steady_clock::now() > deadline) throw std::runtime_error("shm reducer: rank 0 never came up");
        std::this_thread::sleep_for(std::chrono::milliseconds(2));
      }
      for (;;) {  // rank 0 may not have sized it yet
        off_t end = lseek(fd, 0, SEEK_END);
        if (end >= static_cast<off_t>(bytes_)) break;
        if (std::chrono::steady_clock::now() > deadline) throw std::runtime_error("shm reducer: segment never sized");
        std::this_thread::sleep_for(std::chrono::milliseconds(2));
      }
    }
    void* m = mmap(nullptr, bytes_, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (m == MAP_FAILED) throw std::runtime_error("shm reducer: mmap failed");
    base_ = static_cast<char*>(m);
    hdr_ = reinterpret_cast<ShmHeader*>(base_);
    if (rank == 0) {
      hdr_->arrived.store(0);
      hdr_->gen.store(0);
      hdr_->attached.store(0);
      hdr_->world = static_cast<uint32_t>(world);
      hdr_->slot_bytes = kShmSlot;
      hdr_->magic.store(kShmMagic, std::memory_order_release);
    }
    while (hdr_->magic.load(std::memory_order_acquire) != kShmMagic) {
      if (std::chrono::steady_clock::now() > deadline) throw std::runtime_error("shm reducer: header never initialised");
      std::this_thread::sleep_for(std::chrono::milliseconds(1));
    }
    if (hdr_->world != static_cast<uint32_t>(world)) throw std::invalid_argument("shm reducer: world size mismatch");
    hdr_->attached.fetch_add(1);
    barrier();
    if (rank == 0) shm_unlink(name_.c_str());  // everyone is attached: the name is no longer needed
    host_.resize(kShmSlot);
  }
  ~ShmReducer() override {
    if (base_) munmap(base_, bytes_);
  }
  int world() const override { return world_; }
  int rank() const override { return rank_; }
  bool capturable() const override { return false; }

  // host-level collectives (also the CPU test hook gb_shm_allreduce_selftest)
  void allreduce_host(void* data, size_t count, int eb, bool max) {
    const size_t per = kShmSlot / static_cast<size_t>(eb);
    for (size_t off = 0; off < count; off += per) {
      const size_t n = std::min(per, count - off);
      char* mine = slot(rank_);
      std::memcpy(mine, static_cast<char*>(data) + off * eb, n * eb);
      barrier();
      if (eb == 8) fold<double>(static_cast<double*>(data) + off, n, max);
      else fold<float>(static_cast<float*>(data) + off, n, max);
      barrier();
    }
  }
  void broadcast_host(void* data, size_t bytes, int root) {
    for (size_t off = 0; off < bytes; off += kShmSlot) {
      const size_t n = std::min<size_t>(kShmSlot, bytes - off);
      if (rank_ == root) std::memcpy(slot(root), static_cast<char*>(data) + off, n);
      barrier();
      if (rank_ != root) std::memcpy(static_cast<char*>(data) + off, slot(root), n);
      barrier();
    }
  }

  void allreduce(void* buf, size_t count, int eb, bool max, cudaStream_t s) override {
    const size_t bytes = count * static_cast<size_t>(eb);
    if (dev_tmp_.size() < bytes) dev_tmp_.resize(bytes);
    ck(cudaMemcpyAsync(dev_tmp_.data(), buf, bytes, cudaMemcpyDeviceToHost, s), "shm allreduce d2h");
    ck(cudaStreamSynchronize(s), "shm allreduce");
    allreduce_host(dev_tmp_.data(), count, eb, max);
    ck(cudaMemcpyAsync(buf, dev_tmp_.data(), bytes, cudaMemcpyHostToDevice, s), "shm allreduce h2d");
    ck(cudaStreamSynchronize(s), "shm allreduce");
  }
  void broadcast(void* buf, size_t bytes, int root, cudaStream_t s) override {
    if (dev_tmp_.size() < bytes) dev_tmp_.resize(bytes);
    if (rank_ == root) {
      ck(cudaMemcpyAsync(dev_tmp_.data(), buf, bytes, cudaMemcpyDeviceToHost, s), "shm broadcast d2h");
      ck(cudaStreamSynchronize(s), "shm broadcast");
    }
    broadcast_host(dev_tmp_.data(), bytes, root);
    if (rank_ != root) {
      ck(cudaMemcpyAsync(buf, dev_tmp_.data(), bytes, cudaMemcpyHostToDevice, s), "shm broadcast h2d");
      ck(cudaStreamSynchronize(s), "shm broadcast");
    }
  }

 private:
  char* slot(int r) const { return base_ + sizeof(ShmHeader) + 64 + static_cast<size_t>(r) * kShmSlot; }
  template <typename T>
  void fold(T* out, size_t n, bool max) {
    const T* s0 = reinterpret_cast<const T*>(slot(0));
    T* acc = reinterpret_cast<T*>(host_.data());
    std::memcpy(acc, s0, n * sizeof(T));
    for (int r = 1; r < world_; ++r) {
      const T* sr = reinterpret_cast<const T*>(slot(r));
      for (size_t i = 0; i < n; ++i) acc[i] = max ? (sr[i] > acc[i] ? sr[i] : acc[i]) : acc[i] + sr[i];
    }
    std::memcpy(out, acc, n * sizeof(T));
  }
  // sense-free generation barrier over the shared header
  void barrier() {
    const uint32_t g = hdr_->gen.load(std::memory_order_acquire);
    if (hdr_->arrived.fetch_add(1, std::memory_order_acq_rel) + 1 == static_cast<uint32_t>(world_)) {
      hdr_->arrived.store(0, std::memory_order_relaxed);
      hdr_->gen.store(g + 1, std::memory_order_release);
      return;
    }
    const auto deadline = std::chrono::steady_clock::now() + std::chrono::seconds(300);
    for (unsigned spin = 0; hdr_->gen.load(std::memory_order_acquire) == g; ++spin) {
      if (spin < 1024) continue;
      sched_yield();
      if ((spin & 0xffff) == 0 && std::chrono::steady_clock::now() > deadline)
        throw std::runtime_error("shm reducer: barrier timed out (a rank died?)");
    }
  }

  int world_, rank_;
  std::string name_;
  size_t bytes_ = 0;
  char* base_ = nullptr;
  ShmHeader* hdr_ = nullptr;
  std::vector<char> host_, dev_tmp_;
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
  if (kind == 2) {
    uint64_t key = 0;
    std::memcpy(&key, id, sizeof(key));
    return std::make_unique<ShmReducer>(world, rank, key);
  }
  throw std::invalid_argument("unknown reducer kind");
}

void nccl_unique_id(void* out128) {
  NcclApi& api = NcclApi::get();
  ncclUniqueId uid;
  api.check(api.getUniqueId(&uid), "ncclGetUniqueId");
  std::memcpy(out128, &uid, sizeof(uid));
}

// CPU test hook: the shared-memory collectives on host buffers (no CUDA)
void shm_allreduce_selftest(int world, int rank, uint64_t key, double* data, uint64_t n, int max, double* bcast,
                            uint64_t nb) {
  ShmReducer r(world, rank, key);
  r.allreduce_host(data, n, 8, max != 0);
  if (bcast) r.broadcast_host(bcast, nb * sizeof(double), world - 1);
}

}  // namespace gb
