// Generic n-ary factor engine on the device.
//
// Solves graphs of arbitrary vertex sets (additive updates) and factor types
// whose residuals are host-device templates (include/gb_generic_models.hpp),
// with the reference's generic algorithm: Auto (forward dual) Jacobians per
// slot column (factor_descriptor.hpp:610-624), per-vertex CSR accumulation of
// b / diag / block-Jacobi blocks in ascending (factor, slot) order
// (:322-370, :435-482, :710-753), clamp and scaling (linear_system.hpp:67-82),
// block-Jacobi PCG with a matrix-free HVP (pcg.hpp:34-105,
// linear_system.hpp:104-115) and the LM loop (levenberg_marquardt.hpp:115-224).
//
// Unlike the BAL path (every decision on the device inside a CUDA graph),
// this engine keeps the LM/PCG scalar decisions on the host: every reduction
// is a fixed-order block reduction on the device whose per-block partials the
// host sums in order (deterministic). The reference's own engine runs the same
// model traits in oracle/ref_generic.cpp; tests/test_gpu_generic.py compares.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "gb_bal.h"
#include "gb_generic.h"
#include "gb_generic_models.hpp"

namespace gbg {

// ------------------------------------------------------------ dual numbers
template <typename T>
struct Dual {
  T value, deriv;
  __host__ __device__ Dual() : value(0), deriv(0) {}
  __host__ __device__ Dual(T v) : value(v), deriv(0) {}  // NOLINT: implicit like gopt::Dual
  __host__ __device__ Dual(T v, T d) : value(v), deriv(d) {}
};
template <typename T>
__device__ inline Dual<T> operator+(Dual<T> a, Dual<T> b) { return {a.value + b.value, a.deriv + b.deriv}; }
template <typename T>
__device__ inline Dual<T> operator-(Dual<T> a, Dual<T> b) { return {a.value - b.value, a.deriv - b.deriv}; }
template <typename T>
__device__ inline Dual<T> operator*(Dual<T> a, Dual<T> b) {
  return {a.value * b.value, a.value * b.deriv + a.deriv * b.value};
}
template <typename T>
__device__ inline Dual<T> operator/(Dual<T> a, Dual<T> b) {
  const T v = a.value / b.value;
  return {v, (a.deriv - v * b.deriv) / b.value};
}
template <typename T>
__device__ inline Dual<T> operator-(Dual<T> a) { return {-a.value, -a.deriv}; }
template <typename T>
__device__ inline Dual<T> sqrt(Dual<T> a) {
  const T s = ::sqrt(a.value);
  return {s, a.deriv / (T(2) * s)};
}
template <typename T>
__device__ inline Dual<T> sin(Dual<T> a) { return {::sin(a.value), ::cos(a.value) * a.deriv}; }
template <typename T>
__device__ inline Dual<T> cos(Dual<T> a) { return {::cos(a.value), -::sin(a.value) * a.deriv}; }
template <typename T>
__device__ inline T value_of(const Dual<T>& a) { return a.value; }

// ------------------------------------------------------------- factor types
// K slots, R residuals, slot dims, slot -> vertex set, observation and
// constant-data types, residual dispatch (gb_generic_models.hpp).
struct CircleF {
  static constexpr int K = 1, R = 1, SUMD = 2;
  __host__ __device__ static constexpr int dim(int) { return 2; }
  __host__ __device__ static constexpr int vs(int) { return 0; }
  __host__ __device__ static constexpr int pre(int) { return 0; }
  using Obs = gbm::CircleObs;
  using Const = uint8_t;
  template <typename T>
  __device__ static void residual(const T* const* p, const Obs& o, const Const&, T* e) {
    gbm::circle_residual(p[0], o, e);
  }
};
struct StereoF {
  static constexpr int K = 2, R = 3, SUMD = 9;
  __host__ __device__ static constexpr int dim(int s) { return s == 0 ? 6 : 3; }
  __host__ __device__ static constexpr int vs(int s) { return s == 0 ? 0 : 2; }
  __host__ __device__ static constexpr int pre(int s) { return s == 0 ? 0 : 6; }
  using Obs = gbm::StereoObs;
  using Const = gbm::StereoCam;
  template <typename T>
  __device__ static void residual(const T* const* p, const Obs& o, const Const& k, T* e) {
    gbm::stereo_residual(p[0], p[1], o, k, e);
  }
};
struct ImuF {
  static constexpr int K = 4, R = 15, SUMD = 30;
  __host__ __device__ static constexpr int dim(int s) { return (s & 1) ? 9 : 6; }
  __host__ __device__ static constexpr int vs(int s) { return s & 1; }
  __host__ __device__ static constexpr int pre(int s) { return s == 0 ? 0 : (s == 1 ? 6 : (s == 2 ? 15 : 21)); }
  using Obs = gbm::ImuObs;
  using Const = gbm::ImuConst;
  template <typename T>
  __device__ static void residual(const T* const* p, const Obs& o, const Const& k, T* e) {
    gbm::imu_residual(p[0], p[1], p[2], p[3], o, k, e);
  }
};

constexpr int kMaxSets = 3;
constexpr int kBlock = 256;

template <typename FP>
struct VSetDev {
  int dim;
  uint32_t n;
  FP* x;         // [n][dim] current parameters
  FP* xn;        // [n][dim] candidate
  const int64_t* col;  // [n] first column (free) or -1 (fixed)
  int64_t hoff;  // this set's first H block entry (dense dim x dim per vertex)
};
template <typename FP>
struct Sets {
  VSetDev<FP> s[kMaxSets];
};

template <typename FP, typename F>
struct FSetDev {
  uint32_t n;
  const uint32_t* idx;  // [n][K] vertex index within its set
  const typename F::Obs* obs;
  const typename F::Const* cst;  // [n]
  FP* J;   // [n][R * SUMD] slot blocks, row-major (factor_descriptor.hpp:662-670)
  FP* wr;  // [n][R] w * r
  FP* w;   // [n]
  FP* q;   // [n][R] HVP forward values
  // per vertex set: CSR of (factor, slot) items, ascending
  const uint32_t* csr_off[kMaxSets];  // [nv + 1] or null
  const uint32_t* csr_item[kMaxSets];  // factor * K + slot
};

struct LossCfg {
  int huber;
  double delta;
};

template <typename FP>
__device__ inline void loss_eval(LossCfg l, FP s, FP* w, FP* v) {  // loss.hpp:25-40
  if (!l.huber || s <= FP(l.delta * l.delta)) {
    *w = FP(1);
    *v = s;
  } else {
    const FP r = ::sqrt(s);
    *w = FP(l.delta) / r;
    *v = FP(2) * FP(l.delta) * r - FP(l.delta * l.delta);
  }
}

template <typename FP>
__device__ inline FP block_sum(FP v) {
  __shared__ FP sh[32];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[wp] = v;
  __syncthreads();
  FP t = FP(0);
  if (threadIdx.x < 32) {
    t = threadIdx.x < (blockDim.x + 31) / 32 ? sh[threadIdx.x] : FP(0);
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  }
  return t;
}

template <typename FP, typename F>
__device__ inline void gather_params(const Sets<FP>& S, const FSetDev<FP, F>& f, uint32_t i, bool cand, FP* buf) {
#pragma unroll
  for (int s = 0; s < F::K; ++s) {
    const VSetDev<FP>& v = S.s[F::vs(s)];
    const FP* src = (cand ? v.xn : v.x) + static_cast<uint64_t>(F::dim(s)) * f.idx[F::K * i + s];
    for (int k = 0; k < F::dim(s); ++k) buf[F::pre(s) + k] = src[k];
  }
}

// linearize one factor type: residual, loss, Auto Jacobian columns, chi partials
template <typename FP, typename F>
__global__ void __launch_bounds__(kBlock) k_lin(Sets<FP> S, FSetDev<FP, F> f, LossCfg loss, FP* part) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  FP chi = FP(0);
  if (i < f.n) {
    FP buf[F::SUMD];
    gather_params(S, f, i, false, buf);
    const FP* ptr[F::K];
#pragma unroll
    for (int s = 0; s < F::K; ++s) ptr[s] = buf + F::pre(s);
    FP r[F::R];
    F::residual(ptr, f.obs[i], f.cst[i], r);
    FP sq = FP(0);
    for (int k = 0; k < F::R; ++k) sq += r[k] * r[k];
    FP w, v;
    loss_eval(loss, sq, &w, &v);
    chi = v;
    f.w[i] = w;
    for (int k = 0; k < F::R; ++k) f.wr[static_cast<uint64_t>(F::R) * i + k] = w * r[k];
    // Auto: one dual pass per parameter (jacobian_auto_slot)
    Dual<FP> db[F::SUMD];
    const Dual<FP>* dp[F::K];
    for (int k = 0; k < F::SUMD; ++k) db[k] = Dual<FP>(buf[k], FP(0));
#pragma unroll
    for (int s = 0; s < F::K; ++s) dp[s] = db + F::pre(s);
    FP* Ji = f.J + static_cast<uint64_t>(F::R * F::SUMD) * i;
#pragma unroll
    for (int s = 0; s < F::K; ++s) {
      const int d = F::dim(s);
      FP* blk = Ji + F::R * F::pre(s);
      for (int c = 0; c < d; ++c) {
        db[F::pre(s) + c].deriv = FP(1);
        Dual<FP> e[F::R];
        F::residual(dp, f.obs[i], f.cst[i], e);
        for (int row = 0; row < F::R; ++row) blk[row * d + c] = e[row].deriv;
        db[F::pre(s) + c].deriv = FP(0);
      }
    }
  }
  chi = block_sum(chi);
  if (threadIdx.x == 0) part[blockIdx.x] = chi;
}

// chi^2 of one factor type at x (cand = 0) or x_new (cand = 1)
template <typename FP, typename F>
__global__ void __launch_bounds__(kBlock) k_chi(Sets<FP> S, FSetDev<FP, F> f, LossCfg loss, int cand, FP* part) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  FP chi = FP(0);
  if (i < f.n) {
    FP buf[F::SUMD];
    gather_params(S, f, i, cand != 0, buf);
    const FP* ptr[F::K];
#pragma unroll
    for (int s = 0; s < F::K; ++s) ptr[s] = buf + F::pre(s);
    FP r[F::R];
    F::residual(ptr, f.obs[i], f.cst[i], r);
    FP sq = FP(0);
    for (int k = 0; k < F::R; ++k) sq += r[k] * r[k];
    FP w, v;
    loss_eval(loss, sq, &w, &v);
    chi = v;
  }
  chi = block_sum(chi);
  if (threadIdx.x == 0) part[blockIdx.x] = chi;
}

// slot block offset / dim of item (factor a, slot s)
template <typename F>
__device__ inline int slot_prefix(int s) {
  return F::pre(s);
}

// b, diag and the dense H block of every free vertex of set `set` from factor
// type F (accumulate_gradient_and_diagonal + the unscaled precond blocks)
template <typename FP, typename F, int D>
__global__ void __launch_bounds__(kBlock) k_acc(Sets<FP> S, FSetDev<FP, F> f, int set, FP* b, FP* H) {
  const VSetDev<FP>& vs = S.s[set];
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= vs.n || vs.col[v] < 0) return;
  const int64_t col = vs.col[v];
  FP bb[D], hh[D * D];
  for (int k = 0; k < D; ++k) bb[k] = b[col + k];
  FP* Hv = H + vs.hoff + static_cast<int64_t>(D * D) * v;
  for (int k = 0; k < D * D; ++k) hh[k] = Hv[k];
  for (uint32_t q = f.csr_off[set][v]; q < f.csr_off[set][v + 1]; ++q) {
    const uint32_t it = f.csr_item[set][q];
    const uint32_t a = it / F::K;
    const int s = static_cast<int>(it % F::K);
    const FP* blk = f.J + static_cast<uint64_t>(F::R * F::SUMD) * a + F::R * slot_prefix<F>(s);
    const FP* wr = f.wr + static_cast<uint64_t>(F::R) * a;
    const FP w = f.w[a];
    for (int c = 0; c < D; ++c) {
      FP g = FP(0);
      for (int row = 0; row < F::R; ++row) g += blk[row * D + c] * wr[row];
      bb[c] += g;
    }
    for (int c1 = 0; c1 < D; ++c1)
      for (int c2 = 0; c2 < D; ++c2) {
        FP h = FP(0);
        for (int row = 0; row < F::R; ++row) h += blk[row * D + c1] * blk[row * D + c2];
        hh[c1 * D + c2] += w * h;
      }
  }
  for (int k = 0; k < D; ++k) b[col + k] = bb[k];
  for (int k = 0; k < D * D; ++k) Hv[k] = hh[k];
}

// HVP forward of one factor type: q = w J (D p) at the free slot columns
template <typename FP, typename F>
__global__ void __launch_bounds__(kBlock) k_fwd(Sets<FP> S, FSetDev<FP, F> f, const FP* vt) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= f.n) return;
  FP u[F::R];
  for (int k = 0; k < F::R; ++k) u[k] = FP(0);
  const FP* Ji = f.J + static_cast<uint64_t>(F::R * F::SUMD) * i;
#pragma unroll
  for (int s = 0; s < F::K; ++s) {
    const VSetDev<FP>& vs = S.s[F::vs(s)];
    const int64_t col = vs.col[f.idx[F::K * i + s]];
    if (col < 0) continue;
    const int d = F::dim(s);
    const FP* blk = Ji + F::R * F::pre(s);
    for (int row = 0; row < F::R; ++row) {
      FP a = FP(0);
      for (int c = 0; c < d; ++c) a += blk[row * d + c] * vt[col + c];
      u[row] += a;
    }
  }
  const FP w = f.w[i];
  for (int k = 0; k < F::R; ++k) f.q[static_cast<uint64_t>(F::R) * i + k] = w * u[k];
}

// HVP scatter (as a per-vertex gather over the CSR): acc += J_s^T q
template <typename FP, typename F, int D>
__global__ void __launch_bounds__(kBlock) k_back(Sets<FP> S, FSetDev<FP, F> f, int set, FP* acc) {
  const VSetDev<FP>& vs = S.s[set];
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= vs.n || vs.col[v] < 0) return;
  const int64_t col = vs.col[v];
  FP g[D];
  for (int k = 0; k < D; ++k) g[k] = acc[col + k];
  for (uint32_t q = f.csr_off[set][v]; q < f.csr_off[set][v + 1]; ++q) {
    const uint32_t it = f.csr_item[set][q];
    const uint32_t a = it / F::K;
    const int s = static_cast<int>(it % F::K);
    const FP* blk = f.J + static_cast<uint64_t>(F::R * F::SUMD) * a + F::R * slot_prefix<F>(s);
    const FP* qa = f.q + static_cast<uint64_t>(F::R) * a;
    for (int c = 0; c < D; ++c) {
      FP t = FP(0);
      for (int row = 0; row < F::R; ++row) t += blk[row * D + c] * qa[row];
      g[c] += t;
    }
  }
  for (int k = 0; k < D; ++k) acc[col + k] = g[k];
}

// Warp-per-vertex variants for vertices with many incident factors (poses
// seen by ~100 stereo factors): lanes stride over the vertex's items and the
// partial sums meet in a fixed-order butterfly (deterministic).
template <typename FP>
__device__ inline FP warp_allsum(FP v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <typename FP, typename F, int D>
__global__ void __launch_bounds__(kBlock) k_back_w(Sets<FP> S, FSetDev<FP, F> f, int set, FP* acc) {
  const VSetDev<FP>& vs = S.s[set];
  const uint32_t v = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (v >= vs.n || vs.col[v] < 0) return;  // warp-uniform
  FP g[D];
  for (int k = 0; k < D; ++k) g[k] = FP(0);
  for (uint32_t q = f.csr_off[set][v] + lane; q < f.csr_off[set][v + 1]; q += 32) {
    const uint32_t it = f.csr_item[set][q];
    const uint32_t a = it / F::K;
    const int s = static_cast<int>(it % F::K);
    const FP* blk = f.J + static_cast<uint64_t>(F::R * F::SUMD) * a + F::R * F::pre(s);
    const FP* qa = f.q + static_cast<uint64_t>(F::R) * a;
    for (int c = 0; c < D; ++c) {
      FP t = FP(0);
      for (int row = 0; row < F::R; ++row) t += blk[row * D + c] * qa[row];
      g[c] += t;
    }
  }
  const int64_t col = vs.col[v];
  for (int k = 0; k < D; ++k) {
    const FP t = warp_allsum(g[k]);
    if (lane == 0) acc[col + k] += t;
  }
}

template <typename FP, typename F, int D>
__global__ void __launch_bounds__(kBlock) k_acc_w(Sets<FP> S, FSetDev<FP, F> f, int set, FP* b, FP* H) {
  const VSetDev<FP>& vs = S.s[set];
  const uint32_t v = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (v >= vs.n || vs.col[v] < 0) return;  // warp-uniform
  FP bb[D], hh[D * D];
  for (int k = 0; k < D; ++k) bb[k] = FP(0);
  for (int k = 0; k < D * D; ++k) hh[k] = FP(0);
  for (uint32_t q = f.csr_off[set][v] + lane; q < f.csr_off[set][v + 1]; q += 32) {
    const uint32_t it = f.csr_item[set][q];
    const uint32_t a = it / F::K;
    const int s = static_cast<int>(it % F::K);
    const FP* blk = f.J + static_cast<uint64_t>(F::R * F::SUMD) * a + F::R * F::pre(s);
    const FP* wr = f.wr + static_cast<uint64_t>(F::R) * a;
    const FP w = f.w[a];
    for (int c = 0; c < D; ++c) {
      FP gg = FP(0);
      for (int row = 0; row < F::R; ++row) gg += blk[row * D + c] * wr[row];
      bb[c] += gg;
    }
    for (int c1 = 0; c1 < D; ++c1)
      for (int c2 = 0; c2 < D; ++c2) {
        FP h = FP(0);
        for (int row = 0; row < F::R; ++row) h += blk[row * D + c1] * blk[row * D + c2];
        hh[c1 * D + c2] += w * h;
      }
  }
  const int64_t col = vs.col[v];
  FP* Hv = H + vs.hoff + static_cast<int64_t>(D * D) * v;
  for (int k = 0; k < D; ++k) {
    const FP t = warp_allsum(bb[k]);
    if (lane == 0) b[col + k] += t;
  }
  for (int k = 0; k < D * D; ++k) {
    const FP t = warp_allsum(hh[k]);
    if (lane == 0) Hv[k] += t;
  }
}

// HVP forward with one warp per factor and one lane per residual row (wide
// factors such as the 15-row IMU preintegration)
template <typename FP, typename F>
__global__ void __launch_bounds__(kBlock) k_fwd_w(Sets<FP> S, FSetDev<FP, F> f, const FP* vt) {
  const uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int row = threadIdx.x & 31;
  if (i >= f.n || row >= F::R) return;
  const FP* Ji = f.J + static_cast<uint64_t>(F::R * F::SUMD) * i;
  FP u = FP(0);
#pragma unroll
  for (int s = 0; s < F::K; ++s) {
    const VSetDev<FP>& vs = S.s[F::vs(s)];
    const int64_t col = vs.col[f.idx[F::K * i + s]];
    if (col < 0) continue;
    const int d = F::dim(s);
    const FP* blk = Ji + F::R * F::pre(s);
    FP a = FP(0);
    for (int c = 0; c < d; ++c) a += blk[row * d + c] * vt[col + c];
    u += a;
  }
  f.q[static_cast<uint64_t>(F::R) * i + row] = f.w[i] * u;
}

// ------------------------------------------------------------ vector kernels
template <typename FP>
__global__ void k_scale(uint64_t n, const FP* b, const FP* diag, double cmin, double cmax, FP* clamped, FP* D,
                        FP* part_max, int* bad) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  FP gm = FP(0);
  if (i < n) {
    const FP dg = diag[i];
    const FP cl = dg < FP(cmin) ? FP(cmin) : (FP(cmax) < dg ? FP(cmax) : dg);
    clamped[i] = cl;
    D[i] = FP(1) / ::sqrt(cl);
    if (!isfinite(b[i]) || !isfinite(dg)) atomicOr(bad, 1);
    gm = ::fabs(b[i]);
  }
  // block max
  __shared__ FP sh[32];
  for (int o = 16; o > 0; o >>= 1) gm = ::fmax(gm, __shfl_xor_sync(0xffffffffu, gm, o));
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = gm;
  __syncthreads();
  if (threadIdx.x == 0) {
    FP m = FP(0);
    for (int k = 0; k < (int)(blockDim.x + 31) / 32; ++k) m = ::fmax(m, sh[k]);
    part_max[blockIdx.x] = m;
  }
}

template <typename FP>
__global__ void k_dot(uint64_t n, const FP* a, const FP* b, FP* part) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  FP v = i < n ? a[i] * b[i] : FP(0);
  v = block_sum(v);
  if (threadIdx.x == 0) part[blockIdx.x] = v;
}

template <typename FP>
__global__ void k_axpy_vt(uint64_t n, const FP* D, const FP* p, FP* vt) {  // vt = D p
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i < n) vt[i] = D[i] * p[i];
}

template <typename FP>
__global__ void k_hvp_fin(uint64_t n, const FP* D, const FP* p, const FP* acc, double lam, int before, FP* ap) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const FP damp = before ? FP(lam) * D[i] * D[i] : FP(lam);
  ap[i] = damp * p[i] + D[i] * acc[i];
}

// block-Jacobi of one vertex set: B = D H D + damping (linear_system.hpp:120-160),
// Cholesky inverse or the clamped diagonal fallback
template <typename FP, int D>
__global__ void k_precond(Sets<FP> S, int set, const FP* H, const FP* Dv, double lam, int before, double cmin,
                          double cmax, FP* M, int* fallbacks) {
  const VSetDev<FP>& vs = S.s[set];
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= vs.n || vs.col[v] < 0) return;
  const int64_t col = vs.col[v];
  const FP* Hv = H + vs.hoff + static_cast<int64_t>(D * D) * v;
  FP B[D * D], L[D * D];
  for (int i = 0; i < D; ++i)
    for (int j = 0; j < D; ++j) {
      B[i * D + j] = Dv[col + i] * Hv[i * D + j] * Dv[col + j];
      if (i == j) B[i * D + j] += before ? FP(lam) * Dv[col + i] * Dv[col + i] : FP(lam);
    }
  bool ok = true;
  for (int j = 0; j < D && ok; ++j) {  // L L^T = B
    FP s = B[j * D + j];
    for (int k = 0; k < j; ++k) s -= L[j * D + k] * L[j * D + k];
    if (!(s > FP(0))) {
      ok = false;
      break;
    }
    L[j * D + j] = ::sqrt(s);
    for (int i = j + 1; i < D; ++i) {
      FP t = B[i * D + j];
      for (int k = 0; k < j; ++k) t -= L[i * D + k] * L[j * D + k];
      L[i * D + j] = t / L[j * D + j];
    }
  }
  FP* Mv = M + vs.hoff + static_cast<int64_t>(D * D) * v;
  if (ok) {  // inverse column by column: L L^T x = e_c
    for (int c = 0; c < D; ++c) {
      FP y[D];
      for (int i = 0; i < D; ++i) {
        FP t = i == c ? FP(1) : FP(0);
        for (int k = 0; k < i; ++k) t -= L[i * D + k] * y[k];
        y[i] = t / L[i * D + i];
      }
      for (int i = D - 1; i >= 0; --i) {
        FP t = y[i];
        for (int k = i + 1; k < D; ++k) t -= L[k * D + i] * y[k];
        y[i] = t / L[i * D + i];
      }
      for (int i = 0; i < D; ++i) Mv[i * D + c] = y[i];
    }
    for (int i = 0; i < D * D; ++i)
      if (!isfinite(Mv[i])) ok = false;
  }
  if (!ok) {
    for (int i = 0; i < D; ++i)
      for (int j = 0; j < D; ++j) {
        const FP bd = B[i * D + i];
        const FP cl = bd < FP(cmin) ? FP(cmin) : (FP(cmax) < bd ? FP(cmax) : bd);
        Mv[i * D + j] = i == j ? FP(1) / cl : FP(0);
      }
    atomicAdd(fallbacks, 1);
  }
}

// z = M r for one vertex set; r.z and r.r partials per block
template <typename FP, int D>
__global__ void k_apply(Sets<FP> S, int set, const FP* M, const FP* r, FP* z, FP* part_rz, FP* part_rr) {
  const VSetDev<FP>& vs = S.s[set];
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  FP rz = FP(0), rr = FP(0);
  if (v < vs.n && vs.col[v] >= 0) {
    const int64_t col = vs.col[v];
    const FP* Mv = M + vs.hoff + static_cast<int64_t>(D * D) * v;
    for (int i = 0; i < D; ++i) {
      FP t = FP(0);
      for (int j = 0; j < D; ++j) t += Mv[i * D + j] * r[col + j];
      z[col + i] = t;
      rz += r[col + i] * t;
      rr += r[col + i] * r[col + i];
    }
  }
  rz = block_sum(rz);
  rr = block_sum(rr);
  if (threadIdx.x == 0) {
    part_rz[blockIdx.x] = rz;
    part_rr[blockIdx.x] = rr;
  }
}

template <typename FP>
__global__ void k_lincomb(uint64_t n, FP* y, FP a, const FP* x, FP b) {  // y = a y + b x
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i < n) y[i] = a * y[i] + b * x[i];
}

// x_new = x + D (x_pcg * unscale) at the free columns of one set
template <typename FP, int D>
__global__ void k_apply_step(Sets<FP> S, int set, const FP* Dv, const FP* xs, FP unscale) {
  const VSetDev<FP>& vs = S.s[set];
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= vs.n) return;
  const int64_t col = vs.col[v];
  for (int k = 0; k < D; ++k) {
    const FP cur = vs.x[static_cast<uint64_t>(D) * v + k];
    vs.xn[static_cast<uint64_t>(D) * v + k] = col < 0 ? cur : cur + Dv[col + k] * (xs[col + k] * unscale);
  }
}

// ===================================================================== host
#define GCK(x)                                                                                          \
  do {                                                                                                  \
    cudaError_t e__ = (x);                                                                              \
    if (e__ != cudaSuccess) throw std::runtime_error(std::string("CUDA error ") + cudaGetErrorString(e__)); \
  } while (0)

template <typename T>
struct DVec {
  T* p = nullptr;
  size_t n = 0;
  DVec() = default;
  DVec(const DVec&) = delete;
  DVec& operator=(const DVec&) = delete;
  ~DVec() {
    if (p) cudaFree(p);
  }
  T* alloc(size_t k) {
    if (p) cudaFree(p);
    n = k;
    GCK(cudaMalloc(&p, std::max<size_t>(1, k) * sizeof(T)));
    return p;
  }
  T* up(const std::vector<T>& h) {
    alloc(h.size());
    if (!h.empty()) GCK(cudaMemcpy(p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
    return p;
  }
  T* zero() {
    GCK(cudaMemset(p, 0, std::max<size_t>(1, n) * sizeof(T)));
    return p;
  }
};

inline unsigned nblk(uint64_t n) { return static_cast<unsigned>(std::max<uint64_t>(1, (n + kBlock - 1) / kBlock)); }

// fixed-order sum of per-block partials (deterministic)
template <typename FP>
FP sum_parts(const FP* dpart, unsigned n) {
  std::vector<FP> h(n);
  GCK(cudaMemcpy(h.data(), dpart, n * sizeof(FP), cudaMemcpyDeviceToHost));
  FP s = FP(0);
  for (FP v : h) s += v;
  return s;
}

template <typename Fn>
void by_dim(int dim, Fn&& fn) {
  switch (dim) {
    case 2: fn(std::integral_constant<int, 2>{}); break;
    case 3: fn(std::integral_constant<int, 3>{}); break;
    case 6: fn(std::integral_constant<int, 6>{}); break;
    case 9: fn(std::integral_constant<int, 9>{}); break;
    default: throw std::invalid_argument("unsupported vertex dimension");
  }
}

template <typename FP>
struct VSetHost {
  int dim = 0;
  uint32_t n = 0;
  double* user = nullptr;  // AoS binary64, refined in place (VertexDescriptor traits update)
  const uint8_t* fixed = nullptr;
  DVec<FP> x, xn;
  DVec<int64_t> col;
};

template <typename FP, typename F>
struct FSetHost {
  static constexpr int kR = F::R;
  uint32_t n = 0;
  std::vector<uint32_t> hidx;
  DVec<uint32_t> idx;
  DVec<typename F::Obs> obs;
  DVec<typename F::Const> cst;
  DVec<FP> J, wr, w, q;
  DVec<uint32_t> off[kMaxSets], item[kMaxSets];
  uint64_t items[kMaxSets] = {0, 0, 0};

  void upload(const std::vector<typename F::Obs>& o, const std::vector<typename F::Const>& c) {
    n = static_cast<uint32_t>(o.size());
    idx.up(hidx);
    obs.up(o);
    cst.up(c);
    J.alloc(static_cast<size_t>(n) * F::R * F::SUMD);
    wr.alloc(static_cast<size_t>(n) * F::R);
    w.alloc(n);
    q.alloc(static_cast<size_t>(n) * F::R);
  }
  // per vertex set: CSR of (factor, slot) items in ascending order (build_incidence)
  void build_csr(const std::vector<VSetHost<FP>*>& sets) {
    for (int st = 0; st < static_cast<int>(sets.size()); ++st) {
      bool used = false;
      for (int s = 0; s < F::K; ++s) used |= F::vs(s) == st;
      if (!used) continue;
      const uint32_t nv = sets[st]->n;
      std::vector<uint32_t> o(nv + 1, 0), it;
      for (uint32_t a = 0; a < n; ++a)
        for (int s = 0; s < F::K; ++s)
          if (F::vs(s) == st) {
            const uint32_t v = hidx[F::K * a + s];
            if (v >= nv) throw std::invalid_argument("add_factor: slot references unknown vertex id");
            ++o[v + 1];
          }
      for (uint32_t v = 0; v < nv; ++v) o[v + 1] += o[v];
      it.resize(o[nv]);
      std::vector<uint32_t> cur(o.begin(), o.end() - 1);
      for (uint32_t a = 0; a < n; ++a)
        for (int s = 0; s < F::K; ++s)
          if (F::vs(s) == st) it[cur[hidx[F::K * a + s]]++] = F::K * a + s;
      off[st].up(o);
      item[st].up(it);
      items[st] = it.size();
    }
  }
  FSetDev<FP, F> dev() const {
    FSetDev<FP, F> f{};
    f.n = n;
    f.idx = idx.p;
    f.obs = obs.p;
    f.cst = cst.p;
    f.J = J.p;
    f.wr = wr.p;
    f.w = w.p;
    f.q = q.p;
    for (int s = 0; s < kMaxSets; ++s) {
      f.csr_off[s] = off[s].p;
      f.csr_item[s] = item[s].p;
    }
    return f;
  }
};

// per factor type: linearize, accumulate, chi^2, HVP passes
template <typename FP, typename F>
struct FactorOps {
  static FP lin(const Sets<FP>& S, const FSetHost<FP, F>& f, LossCfg l, FP* part) {
    if (!f.n) return FP(0);
    k_lin<FP, F><<<nblk(f.n), kBlock>>>(S, f.dev(), l, part);
    GCK(cudaGetLastError());
    return sum_parts(part, nblk(f.n));
  }
  static FP chi(const Sets<FP>& S, const FSetHost<FP, F>& f, LossCfg l, int cand, FP* part) {
    if (!f.n) return FP(0);
    k_chi<FP, F><<<nblk(f.n), kBlock>>>(S, f.dev(), l, cand, part);
    GCK(cudaGetLastError());
    return sum_parts(part, nblk(f.n));
  }
  // many incident items per vertex: one warp per vertex
  static bool wide(const std::vector<VSetHost<FP>*>& sets, const FSetHost<FP, F>& f, int st) {
    return sets[st]->n && f.items[st] >= 16ull * sets[st]->n;
  }
  static void acc(const Sets<FP>& S, const std::vector<VSetHost<FP>*>& sets, const FSetHost<FP, F>& f, FP* b,
                  FP* H) {
    for (int st = 0; st < static_cast<int>(sets.size()); ++st) {
      if (!f.off[st].p || !f.n) continue;
      by_dim(sets[st]->dim, [&](auto Dc) {
        constexpr int D = decltype(Dc)::value;
        if (D <= 6 && wide(sets, f, st))
          k_acc_w<FP, F, D><<<nblk(32ull * sets[st]->n), kBlock>>>(S, f.dev(), st, b, H);
        else
          k_acc<FP, F, D><<<nblk(sets[st]->n), kBlock>>>(S, f.dev(), st, b, H);
      });
      GCK(cudaGetLastError());
    }
  }
  static void fwd(const Sets<FP>& S, const FSetHost<FP, F>& f, const FP* vt) {
    if (!f.n) return;
    if (F::R >= 8)
      k_fwd_w<FP, F><<<nblk(32ull * f.n), kBlock>>>(S, f.dev(), vt);
    else
      k_fwd<FP, F><<<nblk(f.n), kBlock>>>(S, f.dev(), vt);
    GCK(cudaGetLastError());
  }
  static void back(const Sets<FP>& S, const std::vector<VSetHost<FP>*>& sets, const FSetHost<FP, F>& f, FP* acc) {
    for (int st = 0; st < static_cast<int>(sets.size()); ++st) {
      if (!f.off[st].p || !f.n) continue;
      by_dim(sets[st]->dim, [&](auto Dc) {
        constexpr int D = decltype(Dc)::value;
        if (wide(sets, f, st))
          k_back_w<FP, F, D><<<nblk(32ull * sets[st]->n), kBlock>>>(S, f.dev(), st, acc);
        else
          k_back<FP, F, D><<<nblk(sets[st]->n), kBlock>>>(S, f.dev(), st, acc);
      });
      GCK(cudaGetLastError());
    }
  }
};

template <typename FP, typename F>
FP ops_lin(const Sets<FP>& S, const FSetHost<FP, F>& f, LossCfg l, FP* part) {
  return FactorOps<FP, F>::lin(S, f, l, part);
}
template <typename FP, typename F>
FP ops_chi(const Sets<FP>& S, const FSetHost<FP, F>& f, LossCfg l, int cand, FP* part) {
  return FactorOps<FP, F>::chi(S, f, l, cand, part);
}
template <typename FP, typename F>
void ops_acc(const Sets<FP>& S, const std::vector<VSetHost<FP>*>& sets, const FSetHost<FP, F>& f, FP* b, FP* H) {
  FactorOps<FP, F>::acc(S, sets, f, b, H);
}
template <typename FP, typename F>
void ops_fwd(const Sets<FP>& S, const FSetHost<FP, F>& f, const FP* vt) {
  FactorOps<FP, F>::fwd(S, f, vt);
}
template <typename FP, typename F>
void ops_back(const Sets<FP>& S, const std::vector<VSetHost<FP>*>& sets, const FSetHost<FP, F>& f, FP* acc) {
  FactorOps<FP, F>::back(S, sets, f, acc);
}

template <typename FP>
__global__ void k_diag(Sets<FP> S, int set, int dim, const FP* H, FP* diag) {
  const VSetDev<FP>& vs = S.s[set];
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= vs.n || vs.col[v] < 0) return;
  const FP* Hv = H + vs.hoff + static_cast<int64_t>(dim) * dim * v;
  for (int k = 0; k < dim; ++k) diag[vs.col[v] + k] = Hv[k * dim + k];
}
template <typename FP>
__global__ void k_damp_max(uint64_t n, const FP* D, const FP* cl, FP* part) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  FP m = i < n ? D[i] * D[i] * cl[i] : FP(0);
  __shared__ FP sh[32];
  for (int o = 16; o > 0; o >>= 1) m = ::fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    FP r = FP(0);
    for (int k = 0; k < (int)(blockDim.x + 31) / 32; ++k) r = ::fmax(r, sh[k]);
    part[blockIdx.x] = r;
  }
}
template <typename FP>
__global__ void k_rhs(uint64_t n, const FP* D, const FP* b, FP* rhs) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i < n) rhs[i] = -D[i] * b[i];
}
template <typename FP>
__global__ void k_pred(uint64_t n, const FP* D, const FP* x, const FP* rhs, double lam, int before, FP* part,
                       int* bad) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  FP v = FP(0);
  if (i < n) {
    const FP damp = before ? FP(lam) * D[i] * D[i] : FP(lam);
    v = x[i] * (damp * x[i] + rhs[i]);
    if (!isfinite(D[i] * x[i])) atomicOr(bad, 1);
  }
  v = block_sum(v);
  if (threadIdx.x == 0) part[blockIdx.x] = v;
}

template <typename FP>
FP max_parts(const FP* dpart, unsigned n) {
  std::vector<FP> h(n);
  GCK(cudaMemcpy(h.data(), dpart, n * sizeof(FP), cudaMemcpyDeviceToHost));
  FP m = FP(0);
  for (FP v : h) m = std::max(m, v);
  return m;
}

// The model: vertex sets + factor types. Fs... are the factor types in
// registration order (Graph::add_factor_descriptor).
template <typename FP, typename... Fs>
struct Model {
  std::vector<VSetHost<FP>*> sets;
  std::tuple<FSetHost<FP, Fs>...> fs;
  LossCfg loss{0, 1.0};

  template <typename Fn>
  void each(Fn&& fn) {
    std::apply([&](auto&... f) { (fn(f), ...); }, fs);
  }
};

template <typename FP, typename... Fs>
void lm_solve(Model<FP, Fs...>& m, const gb_lm_config& cfg, gb_solve_report* rep, gb_iteration_record* recs,
              int max_recs) {
  using Clock = std::chrono::steady_clock;
  const auto t_start = Clock::now();
  auto since = [](Clock::time_point t0) { return std::chrono::duration<double>(Clock::now() - t0).count(); };
  // activation: columns of free vertices, sets in registration order (vertex_descriptor.hpp:115-126)
  int64_t N = 0, hsize = 0;
  Sets<FP> S{};
  for (size_t st = 0; st < m.sets.size(); ++st) {
    VSetHost<FP>& v = *m.sets[st];
    std::vector<int64_t> col(v.n);
    std::vector<FP> x(static_cast<size_t>(v.n) * v.dim);
    for (uint32_t i = 0; i < v.n; ++i) {
      col[i] = (v.fixed && v.fixed[i]) ? -1 : N;
      if (col[i] >= 0) N += v.dim;
    }
    for (size_t k = 0; k < x.size(); ++k) x[k] = static_cast<FP>(v.user[k]);
    v.col.up(col);
    v.x.up(x);
    v.xn.alloc(x.size());
    S.s[st] = VSetDev<FP>{v.dim, v.n, v.x.p, v.xn.p, v.col.p, hsize};
    hsize += static_cast<int64_t>(v.dim) * v.dim * v.n;
  }
  int64_t residual_dims = 0, nfactors = 0;
  uint64_t maxn = static_cast<uint64_t>(std::max<int64_t>(N, 1));
  m.each([&](auto& f) {
    f.build_csr(m.sets);
    nfactors += f.n;
    residual_dims += static_cast<int64_t>(f.n) * std::remove_reference_t<decltype(f)>::kR;
    maxn = std::max<uint64_t>(maxn, f.n);
  });
  for (auto* v : m.sets) maxn = std::max<uint64_t>(maxn, v->n);
  DVec<FP> b, diag, clamped, Dv, H, M, vt, acc, rhs, xs, r, z, p, ap, part, part2;
  DVec<int> flag;
  for (auto* d : {&b, &diag, &clamped, &Dv, &vt, &acc, &rhs, &xs, &r, &z, &p, &ap}) d->alloc(N);
  H.alloc(hsize);
  M.alloc(hsize);
  part.alloc(nblk(maxn));
  part2.alloc(nblk(maxn));
  flag.alloc(2);
  const unsigned nbN = nblk(N);
  const bool before = cfg.damping == GB_DAMPING_BEFORE_SCALING;

  bool finite = true;
  FP gmax = FP(0);
  auto linearize = [&]() -> FP {  // LinearSystem::linearize (linear_system.hpp:67-82)
    FP chi = FP(0);
    m.each([&](auto& f) {
      chi += ops_lin(S, f, m.loss, part.p);
    });
    b.zero();
    H.zero();
    m.each([&](auto& f) {
      ops_acc(S, m.sets, f, b.p, H.p);
    });
    diag.zero();
    for (size_t st = 0; st < m.sets.size(); ++st)
      k_diag<FP><<<nblk(m.sets[st]->n), kBlock>>>(S, static_cast<int>(st), m.sets[st]->dim, H.p, diag.p);
    flag.zero();
    k_scale<FP><<<nbN, kBlock>>>(N, b.p, diag.p, cfg.clamp_min, cfg.clamp_max, clamped.p, Dv.p, part2.p, flag.p);
    GCK(cudaGetLastError());
    gmax = max_parts(part2.p, nbN);
    int bad = 0;
    GCK(cudaMemcpy(&bad, flag.p, sizeof(int), cudaMemcpyDeviceToHost));
    finite = std::isfinite(static_cast<double>(chi)) && !bad;
    return chi;
  };
  auto total_error = [&](int cand) -> FP {
    FP chi = FP(0);
    m.each([&](auto& f) {
      chi += ops_chi(S, f, m.loss, cand, part.p);
    });
    return chi;
  };
  auto dot = [&](const FP* x, const FP* y) {
    k_dot<FP><<<nbN, kBlock>>>(N, x, y, part.p);
    return sum_parts(part.p, nbN);
  };
  auto apply_M = [&](const FP* rr, FP* zz, FP* rz) {  // z = M r; returns r.z (r.r unused)
    FP t = FP(0);
    for (size_t st = 0; st < m.sets.size(); ++st) {
      by_dim(m.sets[st]->dim, [&](auto Dc) {
        constexpr int Dd = decltype(Dc)::value;
        k_apply<FP, Dd><<<nblk(m.sets[st]->n), kBlock>>>(S, static_cast<int>(st), M.p, rr, zz, part.p, part2.p);
      });
      t += sum_parts(part.p, nblk(m.sets[st]->n));
    }
    *rz = t;
  };
  auto hvp = [&](const FP* pv, FP* out, FP lam) {  // LinearSystem::hvp
    k_axpy_vt<FP><<<nbN, kBlock>>>(N, Dv.p, pv, vt.p);
    acc.zero();
    m.each([&](auto& f) {
      ops_fwd(S, f, vt.p);
      ops_back(S, m.sets, f, acc.p);
    });
    k_hvp_fin<FP><<<nbN, kBlock>>>(N, Dv.p, pv, acc.p, static_cast<double>(lam), before ? 1 : 0, out);
  };

  if (rep) std::memset(rep, 0, sizeof(*rep));
  FP chi2 = linearize();
  if (!std::isfinite(static_cast<double>(chi2)))
    throw std::runtime_error("levenberg_marquardt: non-finite chi^2 at the initial parameters");
  std::vector<gb_iteration_record> its;
  gb_solve_report R{};
  R.initial_chi2 = R.final_chi2 = static_cast<double>(chi2);
  R.free_dims = N;
  R.active_factors = nfactors;
  R.termination = GB_TERM_MAX_ITERATIONS;
  if (N == 0) {
    R.termination = GB_TERM_NO_FREE_PARAMETERS;
  } else {
    k_damp_max<FP><<<nbN, kBlock>>>(N, Dv.p, clamped.p, part.p);
    FP lambda = FP(cfg.tau) * max_parts(part.p, nbN);
    FP nu = FP(2);
    for (int it = 1; it <= cfg.max_iterations; ++it) {
      const auto t_it = Clock::now();
      gb_iteration_record rec{};
      rec.iteration = it;
      rec.chi2_before = static_cast<double>(chi2);
      rec.lambda = static_cast<double>(lambda);
      if (!finite) {
        rec.chi2_after = rec.chi2_before;
        rec.wall_seconds = since(t_it);
        its.push_back(rec);
        R.termination = GB_TERM_NON_FINITE_LINEARIZATION;
        break;
      }
      if (gmax < FP(cfg.gradient_tolerance)) {
        rec.chi2_after = rec.chi2_before;
        rec.wall_seconds = since(t_it);
        its.push_back(rec);
        R.termination = GB_TERM_GRADIENT_SMALL;
        break;
      }
      // solve_step (linear_system.hpp:185-207): preconditioner, PCG (pcg.hpp:34-105), pred, dx
      flag.zero();
      for (size_t st = 0; st < m.sets.size(); ++st)
        by_dim(m.sets[st]->dim, [&](auto Dc) {
          constexpr int Dd = decltype(Dc)::value;
          k_precond<FP, Dd><<<nblk(m.sets[st]->n), kBlock>>>(S, static_cast<int>(st), H.p, Dv.p,
                                                              static_cast<double>(lambda), before ? 1 : 0,
                                                              cfg.clamp_min, cfg.clamp_max, M.p, flag.p);
        });
      GCK(cudaGetLastError());
      int fb = 0;
      GCK(cudaMemcpy(&fb, flag.p, sizeof(int), cudaMemcpyDeviceToHost));
      rec.precond_fallback_blocks = fb;
      k_rhs<FP><<<nbN, kBlock>>>(N, Dv.p, b.p, rhs.p);
      const FP rhs_norm = std::sqrt(dot(rhs.p, rhs.p));
      int pcg_it = 0;
      bool conv = false;
      double relres = 0.0;
      xs.zero();
      FP unscale = FP(1);
      if (!(rhs_norm > FP(0))) {
        conv = std::isfinite(static_cast<double>(rhs_norm));
      } else {
        const FP scale = cfg.pcg.normalize_rhs ? FP(1) / rhs_norm : FP(1);
        const FP ref_norm = cfg.pcg.normalize_rhs ? FP(1) : rhs_norm;
        GCK(cudaMemcpy(r.p, rhs.p, N * sizeof(FP), cudaMemcpyDeviceToDevice));
        k_lincomb<FP><<<nbN, kBlock>>>(N, r.p, scale, r.p, FP(0));
        FP rho;
        apply_M(r.p, z.p, &rho);
        GCK(cudaMemcpy(p.p, z.p, N * sizeof(FP), cudaMemcpyDeviceToDevice));
        FP res = std::sqrt(dot(r.p, r.p));
        relres = static_cast<double>(res / ref_norm);
        while (pcg_it < cfg.pcg.max_iterations) {
          hvp(p.p, ap.p, lambda);
          const FP pap = dot(p.p, ap.p);
          if (!(pap > FP(0)) || !std::isfinite(static_cast<double>(pap))) {
            conv = false;
            break;
          }
          const FP alpha = rho / pap;
          k_lincomb<FP><<<nbN, kBlock>>>(N, xs.p, FP(1), p.p, alpha);
          k_lincomb<FP><<<nbN, kBlock>>>(N, r.p, FP(1), ap.p, -alpha);
          ++pcg_it;
          res = std::sqrt(dot(r.p, r.p));
          relres = static_cast<double>(res / ref_norm);
          if (!std::isfinite(relres)) {
            conv = false;
            break;
          }
          if (res <= FP(cfg.pcg.tolerance) * ref_norm) {
            conv = true;
            break;
          }
          FP rho_next;
          apply_M(r.p, z.p, &rho_next);
          const FP beta = rho_next / rho;
          rho = rho_next;
          k_lincomb<FP><<<nbN, kBlock>>>(N, p.p, beta, z.p, FP(1));
        }
        unscale = cfg.pcg.normalize_rhs ? rhs_norm : FP(1);
      }
      // x_scaled = xs * unscale: pred and the finiteness of dx = D x_scaled
      k_lincomb<FP><<<nbN, kBlock>>>(N, xs.p, unscale, xs.p, FP(0));
      flag.zero();
      k_pred<FP><<<nbN, kBlock>>>(N, Dv.p, xs.p, rhs.p, static_cast<double>(lambda), before ? 1 : 0, part.p, flag.p);
      const FP pred = sum_parts(part.p, nbN);
      int badx = 0;
      GCK(cudaMemcpy(&badx, flag.p, sizeof(int), cudaMemcpyDeviceToHost));
      const bool step_finite = !badx;
      rec.pcg_iterations = pcg_it;
      rec.pcg_converged = conv ? 1 : 0;
      rec.pcg_relative_residual = relres;
      if (cfg.use_rejection_guard && !conv && relres > cfg.pcg.rejection_ratio * cfg.pcg.tolerance) {
        rec.low_quality_step = 1;
        lambda *= nu;
      }
      FP chi2_new = std::numeric_limits<FP>::quiet_NaN();
      if (step_finite) {
        for (size_t st = 0; st < m.sets.size(); ++st)
          by_dim(m.sets[st]->dim, [&](auto Dc) {
            constexpr int Dd = decltype(Dc)::value;
            k_apply_step<FP, Dd><<<nblk(m.sets[st]->n), kBlock>>>(S, static_cast<int>(st), Dv.p, xs.p, FP(1));
          });
        chi2_new = total_error(1);
      }
      rec.chi2_after = static_cast<double>(chi2_new);
      const bool accepted = std::isfinite(static_cast<double>(chi2_new)) && chi2_new < chi2;
      rec.accepted = accepted ? 1 : 0;
      FP rel = FP(0);
      if (accepted) {
        ++R.accepted_steps;
        const FP gain = pred > FP(0) ? (chi2 - chi2_new) / pred : std::numeric_limits<FP>::infinity();
        const FP g = FP(2) * gain - FP(1);
        lambda *= std::max(FP(1) / FP(3), FP(1) - g * g * g);
        nu = FP(2);
        rel = (chi2 - chi2_new) / chi2;
        for (auto* v : m.sets)  // x <- x_new (the accepted parameters)
          GCK(cudaMemcpy(v->x.p, v->xn.p, v->xn.n * sizeof(FP), cudaMemcpyDeviceToDevice));
        chi2 = linearize();
        R.final_chi2 = static_cast<double>(chi2);
      } else {
        lambda *= nu;
        nu *= FP(2);
        if (cfg.refresh_on_reject) linearize();
      }
      rec.wall_seconds = since(t_it);
      its.push_back(rec);
      if (accepted && static_cast<double>(rel) < cfg.tolerance) {
        R.termination = GB_TERM_TOLERANCE_REACHED;
        break;
      }
      if (static_cast<double>(lambda) > cfg.lambda_max) {
        R.termination = GB_TERM_DAMPING_OVERFLOW;
        break;
      }
    }
  }
  // write back (VertexDescriptor::scatter through Traits::set_parameters)
  for (auto* v : m.sets) {
    std::vector<FP> h(v->x.n);
    GCK(cudaMemcpy(h.data(), v->x.p, h.size() * sizeof(FP), cudaMemcpyDeviceToHost));
    for (size_t k = 0; k < h.size(); ++k) v->user[k] = static_cast<double>(h[k]);
  }
  R.iterations_run = static_cast<int32_t>(its.size());
  R.total_seconds = since(t_start);
  R.residual_dims = residual_dims;
  if (rep) *rep = R;
  if (recs)
    for (int i = 0; i < std::min<int>(max_recs, static_cast<int>(its.size())); ++i) recs[i] = its[i];
}

}  // namespace gbg

// ====================================================================== C ABI
namespace {
thread_local std::string g_gerr;  // per calling thread, like gb_last_error
template <typename Fn>
int gguard(Fn&& f) {
  try {
    f();
    g_gerr.clear();
    return GB_OK;
  } catch (const std::invalid_argument& e) {
    g_gerr = e.what();
    return GB_ERR_INVALID_ARGUMENT;
  } catch (const std::runtime_error& e) {
    g_gerr = e.what();
    return GB_ERR_RUNTIME;
  } catch (const std::exception& e) {
    g_gerr = e.what();
    return GB_ERR_RUNTIME;
  }
}

template <typename FP>
void circle_solve(uint64_t n, double* pts, const double* radius, const gb_lm_config& cfg, gb_solve_report* rep,
                  gb_iteration_record* recs, int max_recs) {
  gbg::Model<FP, gbg::CircleF> m;
  gbg::VSetHost<FP> v;
  v.dim = 2;
  v.n = static_cast<uint32_t>(n);
  v.user = pts;
  m.sets = {&v};
  auto& f = std::get<0>(m.fs);
  std::vector<gbm::CircleObs> obs(n);
  std::vector<uint8_t> cst(n, 0);
  f.hidx.resize(n);
  for (uint64_t i = 0; i < n; ++i) {
    obs[i].radius = radius[i];
    f.hidx[i] = static_cast<uint32_t>(i);
  }
  f.upload(obs, cst);
  gbg::lm_solve(m, cfg, rep, recs, max_recs);
}

template <typename FP>
void vi_solve(uint64_t npose, double* poses, const uint8_t* pose_fixed, uint64_t nvb, double* vbs, uint64_t nlm,
              double* lms, uint64_t nst, const uint32_t* st_idx, const double* st_obs, const double* cam, uint64_t nimu,
              const uint32_t* imu_idx, const double* imu_obs, const double* gravity, const gb_lm_config& cfg,
              gb_solve_report* rep, gb_iteration_record* recs, int max_recs) {
  gbg::Model<FP, gbg::StereoF, gbg::ImuF> m;
  gbg::VSetHost<FP> P, V, X;
  P.dim = 6;
  P.n = static_cast<uint32_t>(npose);
  P.user = poses;
  P.fixed = pose_fixed;
  V.dim = 9;
  V.n = static_cast<uint32_t>(nvb);
  V.user = vbs;
  X.dim = 3;
  X.n = static_cast<uint32_t>(nlm);
  X.user = lms;
  m.sets = {&P, &V, &X};
  auto& sf = std::get<0>(m.fs);
  auto& imf = std::get<1>(m.fs);
  const gbm::StereoCam k{cam[0], cam[1], cam[2], cam[3], cam[4]};
  std::vector<gbm::StereoObs> so(nst);
  std::vector<gbm::StereoCam> sc(nst, k);
  sf.hidx.assign(st_idx, st_idx + 2 * nst);
  for (uint64_t i = 0; i < nst; ++i) so[i] = gbm::StereoObs{st_obs[3 * i], st_obs[3 * i + 1], st_obs[3 * i + 2]};
  sf.upload(so, sc);
  const gbm::ImuConst g{{gravity[0], gravity[1], gravity[2]}};
  std::vector<gbm::ImuObs> io(nimu);
  std::vector<gbm::ImuConst> ic(nimu, g);
  imf.hidx.assign(imu_idx, imu_idx + 4 * nimu);
  for (uint64_t i = 0; i < nimu; ++i) {
    const double* s = imu_obs + 19 * i;
    for (int q = 0; q < 3; ++q) {
      io[i].dp[q] = s[q];
      io[i].dv[q] = s[3 + q];
    }
    for (int q = 0; q < 9; ++q) io[i].dR[q] = s[6 + q];
    io[i].dt = s[15];
  }
  imf.upload(io, ic);
  gbg::lm_solve(m, cfg, rep, recs, max_recs);
}
}  // namespace

extern "C" {

const char* gbg_last_error(void) { return g_gerr.c_str(); }

int gbg_circle_solve(int precision, uint64_t n, double* points, const double* radius, const gb_lm_config* cfg,
                     int device, gb_solve_report* rep, gb_iteration_record* recs, int max_recs) {
  return gguard([&] {
    GCK(cudaSetDevice(device));
    if (precision == GB_FP64)
      circle_solve<double>(n, points, radius, *cfg, rep, recs, max_recs);
    else if (precision == GB_FP32)
      circle_solve<float>(n, points, radius, *cfg, rep, recs, max_recs);
    else
      throw std::invalid_argument("generic path: precision pair must be fp64 or fp32");
  });
}

int gbg_vi_solve(int precision, uint64_t npose, double* poses, const uint8_t* pose_fixed, uint64_t nvb, double* vbs,
                 uint64_t nlm, double* lms, uint64_t nst, const uint32_t* st_idx, const double* st_obs,
                 const double* cam, uint64_t nimu, const uint32_t* imu_idx, const double* imu_obs,
                 const double* gravity, const gb_lm_config* cfg, int device, gb_solve_report* rep,
                 gb_iteration_record* recs, int max_recs) {
  return gguard([&] {
    GCK(cudaSetDevice(device));
    if (precision == GB_FP64)
      vi_solve<double>(npose, poses, pose_fixed, nvb, vbs, nlm, lms, nst, st_idx, st_obs, cam, nimu, imu_idx, imu_obs,
                       gravity, *cfg, rep, recs, max_recs);
    else if (precision == GB_FP32)
      vi_solve<float>(npose, poses, pose_fixed, nvb, vbs, nlm, lms, nst, st_idx, st_obs, cam, nimu, imu_idx, imu_obs,
                      gravity, *cfg, rep, recs, max_recs);
    else
      throw std::invalid_argument("generic path: precision pair must be fp64 or fp32");
  });
}

}  // extern "C"
