// Common device/host helpers: precision pairs, narrowing/widening, and the
// deterministic reductions every kernel uses.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <cstring>

namespace gb {

// Storage-only bfloat16 (reference include/gopt/bfloat16.hpp:12-37).
struct bf16 {
  uint16_t bits;
};

// Arithmetic type backing a storage type (precision.hpp:72-81): bf16 -> float.
template <typename SP>
struct arith_of {
  using type = SP;
};
template <>
struct arith_of<bf16> {
  using type = float;
};
template <typename SP>
using arith_t = typename arith_of<SP>::type;

__host__ __device__ inline float u32_as_f32(uint32_t u) {
#ifdef __CUDA_ARCH__
  return __uint_as_float(u);
#else
  float f;
  std::memcpy(&f, &u, 4);
  return f;
#endif
}
__host__ __device__ inline uint32_t f32_as_u32(float f) {
#ifdef __CUDA_ARCH__
  return __float_as_uint(f);
#else
  uint32_t u;
  std::memcpy(&u, &f, 4);
  return u;
#endif
}

// RNE narrowing identical to bfloat16::round_from (bfloat16.hpp:25-33),
// including the quiet-NaN-with-sign encoding.
__host__ __device__ inline uint16_t bf16_round(float f) {
  const uint32_t u = f32_as_u32(f);
  if (f != f) return static_cast<uint16_t>(((u >> 16) & 0x8000u) | 0x7FC0u);
  const uint32_t bias = 0x7FFFu + ((u >> 16) & 1u);
  return static_cast<uint16_t>((u + bias) >> 16);
}

// narrow<SP>(x): precision.hpp:86-94 (bf16 goes through float first).
template <typename SP>
struct Narrow {
  template <typename From>
  __host__ __device__ static SP apply(From x) {
    return static_cast<SP>(x);
  }
};
template <>
struct Narrow<bf16> {
  template <typename From>
  __host__ __device__ static bf16 apply(From x) {
    return bf16{bf16_round(static_cast<float>(x))};
  }
};
template <typename SP, typename From>
__host__ __device__ inline SP narrow(From x) {
  return Narrow<SP>::apply(x);
}

// widen<To>(x): precision.hpp:97-100.
template <typename To>
__host__ __device__ inline To widen(double x) {
  return static_cast<To>(x);
}
template <typename To>
__host__ __device__ inline To widen(float x) {
  return static_cast<To>(x);
}
template <typename To>
__host__ __device__ inline To widen(bf16 x) {
  return static_cast<To>(u32_as_f32(static_cast<uint32_t>(x.bits) << 16));
}

// Explicitly rounded multiply / fused multiply-add: the factored Jacobian
// store rebuilds J entries in the HVP with exactly the
// operations linearize used, so these must not be left to FMA contraction.
__device__ inline double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ inline float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ inline double fma_rn(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ inline float fma_rn(float a, float b, float c) { return __fmaf_rn(a, b, c); }

template <typename T>
__host__ __device__ inline bool is_finite(T x) {
  return isfinite(x);
}

// ---- deterministic reductions ------------------------------------------------
// Every reduction below has a fixed association order for a fixed launch
// shape, so results are bitwise reproducible run to run (the reference's
// worker-count-independence contract, parallel.hpp:9-12).

template <typename T>
__device__ inline T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <typename T>
__device__ inline T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide sum; every thread gets the result. scratch: >= 32 T.
template <typename T>
__device__ inline T block_sum(T v, T* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  T r = lane < nw ? scratch[lane] : T(0);
  r = warp_sum(r);
  return r;
}
template <typename T>
__device__ inline T block_max(T v, T* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  T r = lane < nw ? scratch[lane] : T(-INFINITY);
  r = warp_max(r);
  return r;
}

// "Last block done": call after this block published its partial (all
// threads). Returns true in exactly one block, after every block's partial
// is visible. The counter is reset for the next launch.
__device__ inline bool last_block(unsigned* counter) {
  __shared__ bool is_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned t = atomicAdd(counter, 1u);
    is_last = (t == gridDim.x - 1);
    if (is_last) *counter = 0;
  }
  __syncthreads();
  if (is_last) __threadfence();
  return is_last;
}

// Sum of n partials in a fixed order by one block: each thread keeps four
// independent accumulators over a fixed stride pattern (loads pipeline), then
// a fixed tree. ld.cg: the partials were written by other blocks of the same
// launch and are visible in L2 after their __threadfence.
template <typename T>
__device__ inline T ldcg(const T* p) {
  return __ldcg(p);
}
template <typename T>
__device__ inline T reduce_partials(const T* p, uint32_t n, T* scratch) {
  T a0 = T(0), a1 = T(0), a2 = T(0), a3 = T(0);
  const uint32_t st = blockDim.x;
  uint32_t i = threadIdx.x;
  for (; i + 3 * st < n; i += 4 * st) {
    a0 += ldcg(p + i);
    a1 += ldcg(p + i + st);
    a2 += ldcg(p + i + 2 * st);
    a3 += ldcg(p + i + 3 * st);
  }
  for (; i < n; i += st) a0 += ldcg(p + i);
  return block_sum((a0 + a1) + (a2 + a3), scratch);
}
template <typename T>
__device__ inline T reduce_partials_max(const T* p, uint32_t n, T* scratch) {
  T a0 = T(-INFINITY), a1 = T(-INFINITY);
  const uint32_t st = blockDim.x;
  uint32_t i = threadIdx.x;
  for (; i + st < n; i += 2 * st) {
    a0 = fmax(a0, ldcg(p + i));
    a1 = fmax(a1, ldcg(p + i + st));
  }
  for (; i < n; i += st) a0 = fmax(a0, ldcg(p + i));
  return block_max(fmax(a0, a1), scratch);
}
__device__ inline int reduce_flags_and(const int* p, uint32_t n) {
  int f = 1;
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) f &= __ldcg(p + i);
  return __syncthreads_and(f);
}
__device__ inline int reduce_flags_or(const int* p, uint32_t n) {
  int f = 0;
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) f |= __ldcg(p + i);
  return __syncthreads_or(f);
}

}  // namespace gb
