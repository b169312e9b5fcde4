// Streaming microbenchmark for the pipelined-HVP design space: a persistent
// CTA per SM pulls a large buffer through a ring of shared-memory stages with
// 1-D bulk async copies, varying the stage size, the stage count and the
// number of copies per stage. Prints GB/s per configuration.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_bench tools/tma_bench.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

__device__ inline uint32_t sa(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void __launch_bounds__(64, 1) k_stream(const char* src, uint64_t chunk_bytes, uint64_t nchunks, int stages,
                                                  int copies, unsigned long long* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + stages * chunk_bytes);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&full[s])), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  unsigned long long acc = 0;
  const uint32_t piece = static_cast<uint32_t>(chunk_bytes / copies);
  // warp 0 lane 0..: producer; warp 1: consumer (touches one word per chunk)
  uint32_t i = 0;
  for (uint64_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++i) {
    const int s = i % stages;
    unsigned char* st = sm + s * chunk_bytes;
    if (i >= static_cast<uint32_t>(stages)) {
      // wait for the previous use of this stage to complete (consumer reads it below)
      asm volatile(
          "{\n .reg .pred P;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n @!P bra W_%=;\n}" ::"r"(
              sa(&full[s])),
          "r"(((i / stages) - 1) & 1)
          : "memory");
    }
    __syncthreads();
    if (warp == 0) {
      if (lane == 0)
        asm volatile("{\n .reg .b64 t;\n mbarrier.arrive.expect_tx.shared::cta.b64 t, [%0], %1;\n}" ::"r"(sa(&full[s])),
                     "r"(static_cast<uint32_t>(chunk_bytes))
                     : "memory");
      __syncwarp();
      for (int q = lane; q < copies; q += 32)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                sa(st + q * piece)),
            "l"(src + c * chunk_bytes + q * piece), "r"(piece), "r"(sa(&full[s]))
            : "memory");
    }
    if (warp == 1 && i >= static_cast<uint32_t>(stages) - 1) {
      // consume the oldest outstanding stage
      const uint32_t j = i - (stages - 1);
      const int sj = j % stages;
      asm volatile(
          "{\n .reg .pred P;\nV_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n @!P bra V_%=;\n}" ::"r"(
              sa(&full[sj])),
          "r"((j / stages) & 1)
          : "memory");
      acc += sm[sj * chunk_bytes + lane];
    }
  }
  // drain
  if (warp == 1) {
    const uint32_t first = i >= static_cast<uint32_t>(stages) - 1 ? i - (stages - 1) : 0;
    for (uint32_t j = first; j < i; ++j) {
      const int sj = j % stages;
      asm volatile(
          "{\n .reg .pred P;\nX_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n @!P bra X_%=;\n}" ::"r"(
              sa(&full[sj])),
          "r"((j / stages) & 1)
          : "memory");
      acc += sm[sj * chunk_bytes + lane];
    }
  }
  if (acc == 0xdeadbeef) *sink = acc;
}

int main() {
  const uint64_t total = 4ull << 30;
  char* buf;
  unsigned long long* sink;
  cudaMalloc(&buf, total + (1 << 20));
  cudaMalloc(&sink, 8);
  cudaMemset(buf, 1, total);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  struct Cfg {
    uint64_t chunk;
    int stages, copies;
  };
  std::vector<Cfg> cfgs = {{65536, 2, 1},  {65536, 2, 16}, {65536, 2, 32}, {65536, 2, 64}, {65536, 2, 128},
                           {98304, 2, 24}, {98304, 2, 48}, {98304, 2, 96}, {32768, 4, 8},  {32768, 4, 32},
                           {16384, 8, 4},  {49152, 4, 12}};
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (auto c : cfgs) {
    const uint64_t n = total / c.chunk;
    const size_t smem = c.stages * c.chunk + 8 * c.stages;
    if (smem > 227 * 1024) continue;
    k_stream<<<sms, 64, smem>>>(buf, c.chunk, n, c.stages, c.copies, sink);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) k_stream<<<sms, 64, smem>>>(buf, c.chunk, n, c.stages, c.copies, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("chunk %6llu B x %2d stages, %2d copies/chunk: %7.1f GB/s  (%s)\n", (unsigned long long)c.chunk, c.stages,
           c.copies, 5.0 * n * c.chunk / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
