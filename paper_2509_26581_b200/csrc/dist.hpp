// Collectives for the sharded solve: the solver only needs a
// sum/max allreduce of small FP buffers (camera-sized vectors and PCG
// scalars) and a broadcast for the final point gather.
//
//   NcclReducer      one process per GPU, NCCL over NVLink/NVSwitch; NCCL is
//                    loaded at runtime (dlopen libnccl.so.2, the copy torch
//                    already loaded when present) and its calls are captured
//                    into the per-iteration CUDA graph.
//   LoopbackReducer  K shards inside ONE process on ONE GPU (host threads,
//                    eager launches, host rendezvous per collective). Lets the
//                    sharded path be tested on a single device; results are
//                    reduced in rank order like a deterministic allreduce.
//   ShmReducer       one PROCESS per rank on one host (any GPUs, also all on
//                    the same device): POSIX shared memory, host barriers,
//                    rank-order sums. Lets the sharded path run as real
//                    separate processes where NCCL cannot (one GPU).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <memory>

namespace gb {

class Reducer {
 public:
  virtual ~Reducer() = default;
  virtual int world() const = 0;
  virtual int rank() const = 0;
  virtual bool capturable() const = 0;
  // in place; elem_bytes 8 (double) or 4 (float)
  virtual void allreduce(void* buf, size_t count, int elem_bytes, bool max, cudaStream_t s) = 0;
  virtual void broadcast(void* buf, size_t bytes, int root, cudaStream_t s) = 0;
};

// kind 0: NCCL, id = 128-byte ncclUniqueId; kind 1: loopback, id = uint64 group
// key; kind 2: shared memory, id = uint64 segment key
std::unique_ptr<Reducer> make_reducer(int kind, int world, int rank, const void* id);
// the shared-memory collectives on host buffers (CPU test hook): sum/max
// allreduce of data[n], then a broadcast of bcast[nb] from rank world-1
void shm_allreduce_selftest(int world, int rank, uint64_t key, double* data, uint64_t n, int max, double* bcast,
                            uint64_t nb);
// ncclGetUniqueId through the runtime-loaded NCCL (128 bytes)
void nccl_unique_id(void* out128);

}  // namespace gb
