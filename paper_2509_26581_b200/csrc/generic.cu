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
// Like the BAL path, every LM / PCG decision runs on the device: the scalars
// live in a device GState, each reduction is a fixed-order block reduction
// whose per-block partials a one-block decision kernel folds in order
// (deterministic), every kernel is gated by the state's flags, and one LM
// iteration (pcg.max_iterations unrolled PCG steps) is captured once into a
// CUDA graph and replayed; the host only polls a termination flag one
// iteration behind. The reference's own engine runs the same model traits in
// oracle/ref_generic.cpp; tests/test_gpu_generic.py compares.
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
__global__ void __launch_bounds__(kBlock) k_lin(const int* on, Sets<FP> S, FSetDev<FP, F> f, LossCfg loss, FP* part) {
  if (on && !*on) return;  // device-side gate (LM / PCG state)
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
__global__ void __launch_bounds__(kBlock) k_chi(const int* on, Sets<FP> S, FSetDev<FP, F> f, LossCfg loss, int cand, FP* part) {
  if (on && !*on) return;  // device-side gate (LM / PCG state)
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
__global__ void __launch_bounds__(kBlock) k_acc(const int* on, Sets<FP> S, FSetDev<FP, F> f, int set, FP* b, FP* H) {
  if (on && !*on) return;  // device-side gate (LM / PCG state)
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
__global__ void __launch_bounds__(kBlock) k_fwd(const int* on, Sets<FP> S, FSetDev<FP, F> f, const FP* vt) {
  if (on && !*on) return;  // device-side gate (LM / PCG state)
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
__global__ void __launch_bounds__(kBlock) k_back(const int* on, Sets<FP> S, FSetDev<FP, F> f, int set, FP* acc) {
  if (on && !*on) return;  // device-side gate (LM / PCG state)
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
__global__ void __launch_bounds__(kBlock) k_back_w(const int* on, Sets<FP> S, FSetDev<FP, F> f, int set, FP* acc) {
  if (on && !*on) return;  // device-side gate (LM / PCG state)
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
__global__ void __launch_bounds__(kBlock) k_acc_w(const int* on, Sets<FP> S, FSetDev<FP, F> f, int set, FP* b, FP* H) {
  if (on && !*on) return;  // device-side gate (LM / PCG state)
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
__global__ void __launch_bounds__(kBlock) k_fwd_w(const int* on, Sets<FP> S, FSetDev<FP, F> f, const FP* vt) {
  if (on && !*on) return;  // device-side gate (LM / PCG state)
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

// ------------------------------------------------------------ device state
// Every LM / PCG scalar lives here; the decisions are one-block kernels, so an
// LM iteration is a fixed kernel sequence (captured once into a CUDA graph,
// like the BAL path) and the host never waits on a reduction.
template <typename FP>
struct GState {
  FP chi2, lambda, nu, gmax, rhs_norm, scale, ref_norm, unscale, rho, alpha, pred;
  double relres, final_chi2;
  int it, terminated, termination, accepted_steps;
  // gates: iteration running, PCG running, step finite (candidate evaluated),
  // accepted (commit), linearize now
  int iter_active, pcg_active, step_ok, accepted, do_lin;
  int finite, pcg_it, pcg_conv, fallbacks, bad, badx;
};

// LM configuration as the device reads it
struct GCfg {
  int max_it, pcg_max_it, normalize_rhs, use_guard, refresh_on_reject, before;
  double tol, grad_tol, lambda_max, tau, pcg_tol, pcg_ratio, cmin, cmax;
};

// up to 4 partial-sum segments folded in order
template <typename FP>
struct Segs {
  const FP* p[4];
  unsigned n[4];
  int count;
};

// fixed-order fold of per-block partials inside ONE block (deterministic):
// strided per-thread sums, then a shared-memory tree; result on every thread
template <typename FP>
__device__ FP block_fold(const FP* p, unsigned n, bool mx) {
  __shared__ FP sh[kBlock];
  FP acc = FP(0);
  for (unsigned i = threadIdx.x; i < n; i += blockDim.x) acc = mx ? ::fmax(acc, p[i]) : acc + p[i];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int o = kBlock / 2; o > 0; o >>= 1) {
    if (static_cast<int>(threadIdx.x) < o)
      sh[threadIdx.x] = mx ? ::fmax(sh[threadIdx.x], sh[threadIdx.x + o]) : sh[threadIdx.x] + sh[threadIdx.x + o];
    __syncthreads();
  }
  const FP r = sh[0];
  __syncthreads();
  return r;
}
template <typename FP>
__device__ FP fold_segs(const Segs<FP>& s) {
  FP t = FP(0);
  for (int k = 0; k < s.count; ++k) t += block_fold(s.p[k], s.n[k], false);
  return t;
}

// ------------------------------------------------------------ vector kernels
#define GGATE \
  if (on && !*on) return
template <typename FP>
__global__ void k_scale(const int* on, uint64_t n, const FP* b, const FP* diag, double cmin, double cmax, FP* clamped,
                        FP* D, FP* part_max, int* bad) {
  GGATE;
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
__global__ void k_dot(const int* on, uint64_t n, const FP* a, const FP* b, FP* part) {
  GGATE;
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  FP v = i < n ? a[i] * b[i] : FP(0);
  v = block_sum(v);
  if (threadIdx.x == 0) part[blockIdx.x] = v;
}

template <typename FP>
__global__ void k_axpy_vt(const int* on, uint64_t n, const FP* D, const FP* p, FP* vt) {  // vt = D p
  GGATE;
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i < n) vt[i] = D[i] * p[i];
}

template <typename FP>
__global__ void k_hvp_fin(const int* on, uint64_t n, const FP* D, const FP* p, const FP* acc, const GState<FP>* st,
                          int before, FP* ap) {
  GGATE;
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const FP lam = st->lambda;
  const FP damp = before ? lam * D[i] * D[i] : lam;
  ap[i] = damp * p[i] + D[i] * acc[i];
}

template <typename T>
__global__ void k_fill(const int* on, uint64_t n, T* y, T v) {
  GGATE;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    y[i] = v;
}
template <typename T>
__global__ void k_copy(const int* on, uint64_t n, T* y, const T* x) {
  GGATE;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    y[i] = x[i];
}

// block-Jacobi of one vertex set: B = D H D + damping (linear_system.hpp:120-160),
// Cholesky inverse or the clamped diagonal fallback
template <typename FP, int D>
__global__ void k_precond(const int* on, Sets<FP> S, int set, const FP* H, const FP* Dv, const GState<FP>* st,
                          int before, double cmin, double cmax, FP* M, int* fallbacks) {
  GGATE;
  const VSetDev<FP>& vs = S.s[set];
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= vs.n || vs.col[v] < 0) return;
  const FP lam = st->lambda;
  const int64_t col = vs.col[v];
  const FP* Hv = H + vs.hoff + static_cast<int64_t>(D * D) * v;
  FP B[D * D], L[D * D];
  for (int i = 0; i < D; ++i)
    for (int j = 0; j < D; ++j) {
      B[i * D + j] = Dv[col + i] * Hv[i * D + j] * Dv[col + j];
      if (i == j) B[i * D + j] += before ? lam * Dv[col + i] * Dv[col + i] : lam;
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

// z = M r for one vertex set; r.z partials per block
template <typename FP, int D>
__global__ void k_apply(const int* on, Sets<FP> S, int set, const FP* M, const FP* r, FP* z, FP* part_rz) {
  GGATE;
  const VSetDev<FP>& vs = S.s[set];
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  FP rz = FP(0);
  if (v < vs.n && vs.col[v] >= 0) {
    const int64_t col = vs.col[v];
    const FP* Mv = M + vs.hoff + static_cast<int64_t>(D * D) * v;
    for (int i = 0; i < D; ++i) {
      FP t = FP(0);
      for (int j = 0; j < D; ++j) t += Mv[i * D + j] * r[col + j];
      z[col + i] = t;
      rz += r[col + i] * t;
    }
  }
  rz = block_sum(rz);
  if (threadIdx.x == 0) part_rz[blockIdx.x] = rz;
}

// r = scale * rhs (pcg.hpp:49-54: multiply by the reciprocal)
template <typename FP>
__global__ void k_init_r(const int* on, uint64_t n, const GState<FP>* st, const FP* rhs, FP* r) {
  GGATE;
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i < n) r[i] = st->scale * rhs[i] + FP(0) * rhs[i];
}
// x += alpha p; r -= alpha ap (pcg.hpp:78-80)
template <typename FP>
__global__ void k_update_xr(const int* on, uint64_t n, const GState<FP>* st, const FP* p, const FP* ap, FP* x, FP* r) {
  GGATE;
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const FP a = st->alpha;
  x[i] = FP(1) * x[i] + a * p[i];
  r[i] = FP(1) * r[i] + (-a) * ap[i];
}
// p = beta p + z
template <typename FP>
__global__ void k_dir(const int* on, uint64_t n, const FP* beta, const FP* z, FP* p) {
  GGATE;
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i < n) p[i] = *beta * p[i] + FP(1) * z[i];
}
// x *= unscale (x_scaled = x_pcg * ||rhs||)
template <typename FP>
__global__ void k_unscale(const int* on, uint64_t n, const GState<FP>* st, FP* x) {
  GGATE;
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i < n) x[i] = st->unscale * x[i] + FP(0) * x[i];
}

// x_new = x + D x_scaled at the free columns of one set
template <typename FP, int D>
__global__ void k_apply_step(const int* on, Sets<FP> S, int set, const FP* Dv, const FP* xs) {
  GGATE;
  const VSetDev<FP>& vs = S.s[set];
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= vs.n) return;
  const int64_t col = vs.col[v];
  for (int k = 0; k < D; ++k) {
    const FP cur = vs.x[static_cast<uint64_t>(D) * v + k];
    vs.xn[static_cast<uint64_t>(D) * v + k] = col < 0 ? cur : cur + Dv[col + k] * (xs[col + k] * FP(1));
  }
}

template <typename FP>
__global__ void k_diag(const int* on, Sets<FP> S, int set, int dim, const FP* H, FP* diag) {
  GGATE;
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
__global__ void k_rhs(const int* on, uint64_t n, const FP* D, const FP* b, FP* rhs) {
  GGATE;
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i < n) rhs[i] = -D[i] * b[i];
}
template <typename FP>
__global__ void k_pred(const int* on, uint64_t n, const FP* D, const FP* x, const FP* rhs, const GState<FP>* st,
                       int before, FP* part, int* bad) {
  GGATE;
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  FP v = FP(0);
  if (i < n) {
    const FP lam = st->lambda;
    const FP damp = before ? lam * D[i] * D[i] : lam;
    v = x[i] * (damp * x[i] + rhs[i]);
    if (!isfinite(D[i] * x[i])) atomicOr(bad, 1);
  }
  v = block_sum(v);
  if (threadIdx.x == 0) part[blockIdx.x] = v;
}

// ------------------------------------------------------- decision kernels
// (one block each; every thread takes part in the folds, thread 0 decides)

// levenberg_marquardt.hpp:149-169: record start, the non-finite and gradient checks
template <typename FP>
__global__ void k_g_iter_begin(GState<FP>* st, gb_iteration_record* recs, GCfg c) {
  if (threadIdx.x != 0) return;
  st->accepted = 0;
  st->step_ok = 0;
  st->do_lin = 0;
  st->pcg_active = 0;
  if (st->terminated || st->it >= c.max_it) {
    st->iter_active = 0;
    return;
  }
  const int it = ++st->it;
  gb_iteration_record& r = recs[it - 1];
  r = gb_iteration_record{};
  r.iteration = it;
  r.chi2_before = static_cast<double>(st->chi2);
  r.lambda = static_cast<double>(st->lambda);
  if (!st->finite || st->gmax < FP(c.grad_tol)) {
    r.chi2_after = r.chi2_before;
    st->termination = !st->finite ? GB_TERM_NON_FINITE_LINEARIZATION : GB_TERM_GRADIENT_SMALL;
    st->terminated = 1;
    st->iter_active = 0;
    return;
  }
  st->iter_active = 1;
  st->fallbacks = 0;
  st->badx = 0;
  st->pcg_it = 0;
  st->pcg_conv = 0;
  st->relres = 0.0;
  st->unscale = FP(1);
}

// pcg.hpp:43-57: rhs norm, scaling
template <typename FP>
__global__ void k_g_pcg_begin(GState<FP>* st, const FP* part, unsigned n, GCfg c) {
  if (!st->iter_active) return;
  const FP nrm = ::sqrt(block_fold(part, n, false));
  if (threadIdx.x != 0) return;
  st->rhs_norm = nrm;
  if (!(nrm > FP(0))) {
    st->pcg_conv = isfinite(nrm) ? 1 : 0;
    st->pcg_active = 0;
    st->unscale = FP(1);
    return;
  }
  st->scale = c.normalize_rhs ? FP(1) / nrm : FP(1);
  st->ref_norm = c.normalize_rhs ? FP(1) : nrm;
  st->unscale = c.normalize_rhs ? nrm : FP(1);
  st->pcg_active = 1;
}

// rho = r.z (sets in order), res = |r| (pcg.hpp:58-64)
template <typename FP>
__global__ void k_g_rho(GState<FP>* st, Segs<FP> rz, const FP* part_rr, unsigned n) {
  if (!st->pcg_active) return;
  const FP rho = fold_segs(rz);
  const FP rr = block_fold(part_rr, n, false);
  if (threadIdx.x != 0) return;
  st->rho = rho;
  st->relres = static_cast<double>(::sqrt(rr) / st->ref_norm);
}

// pcg.hpp:70-77: pAp, breakdown check, alpha
template <typename FP>
__global__ void k_g_pap(GState<FP>* st, const FP* part, unsigned n) {
  if (!st->pcg_active) return;
  const FP pap = block_fold(part, n, false);
  if (threadIdx.x != 0) return;
  if (!(pap > FP(0)) || !isfinite(pap)) {
    st->pcg_conv = 0;
    st->pcg_active = 0;
    return;
  }
  st->alpha = st->rho / pap;
}

// pcg.hpp:81-88: iteration count, residual, convergence
template <typename FP>
__global__ void k_g_res(GState<FP>* st, const FP* part, unsigned n, GCfg c) {
  if (!st->pcg_active) return;
  const FP res = ::sqrt(block_fold(part, n, false));
  if (threadIdx.x != 0) return;
  ++st->pcg_it;
  st->relres = static_cast<double>(res / st->ref_norm);
  if (!isfinite(st->relres)) {
    st->pcg_conv = 0;
    st->pcg_active = 0;
  } else if (res <= FP(c.pcg_tol) * st->ref_norm) {
    st->pcg_conv = 1;
    st->pcg_active = 0;
  } else if (st->pcg_it >= c.pcg_max_it) {
    st->pcg_active = 0;  // max_iterations: the trailing direction update changes no output
  }
}

// pcg.hpp:89-93: rho' = r.z, beta (then p = z + beta p)
template <typename FP>
__global__ void k_g_beta(GState<FP>* st, Segs<FP> rz, FP* beta_out) {
  if (!st->pcg_active) return;
  const FP rho_next = fold_segs(rz);
  if (threadIdx.x != 0) return;
  *beta_out = rho_next / st->rho;
  st->rho = rho_next;
}

// linear_system.hpp:198-206 pred + finiteness, levenberg_marquardt.hpp:170-178 guard
template <typename FP>
__global__ void k_g_step(GState<FP>* st, gb_iteration_record* recs, const FP* part, unsigned n, GCfg c) {
  if (!st->iter_active) return;
  const FP pred = block_fold(part, n, false);
  if (threadIdx.x != 0) return;
  st->pred = pred;
  gb_iteration_record& r = recs[st->it - 1];
  r.pcg_iterations = st->pcg_it;
  r.pcg_converged = st->pcg_conv;
  r.pcg_relative_residual = st->relres;
  r.precond_fallback_blocks = st->fallbacks;
  if (c.use_guard && !st->pcg_conv && st->relres > c.pcg_ratio * c.pcg_tol) {
    r.low_quality_step = 1;
    st->lambda *= st->nu;
  }
  st->step_ok = st->badx ? 0 : 1;
}

// levenberg_marquardt.hpp:179-219: candidate chi^2, accept / reject, Nielsen,
// termination (the re-linearization itself follows, gated on do_lin)
template <typename FP>
__global__ void k_g_decide(GState<FP>* st, gb_iteration_record* recs, Segs<FP> chi, GCfg c) {
  if (!st->iter_active) return;
  const FP s = fold_segs(chi);
  if (threadIdx.x != 0) return;
  const FP chi2_new = st->step_ok ? s : FP(NAN);
  gb_iteration_record& r = recs[st->it - 1];
  r.chi2_after = static_cast<double>(chi2_new);
  const bool acc = isfinite(chi2_new) && chi2_new < st->chi2;
  r.accepted = acc ? 1 : 0;
  st->accepted = acc ? 1 : 0;
  FP rel = FP(0);
  if (acc) {
    ++st->accepted_steps;
    const FP gain = st->pred > FP(0) ? (st->chi2 - chi2_new) / st->pred : FP(INFINITY);
    const FP g = FP(2) * gain - FP(1);
    st->lambda *= ::fmax(FP(1) / FP(3), FP(1) - g * g * g);
    st->nu = FP(2);
    rel = (st->chi2 - chi2_new) / st->chi2;
    st->do_lin = 1;
  } else {
    st->lambda *= st->nu;
    st->nu *= FP(2);
    st->do_lin = c.refresh_on_reject ? 1 : 0;
  }
  if (acc && static_cast<double>(rel) < c.tol) {
    st->termination = GB_TERM_TOLERANCE_REACHED;
    st->terminated = 1;
  } else if (static_cast<double>(st->lambda) > c.lambda_max) {
    st->termination = GB_TERM_DAMPING_OVERFLOW;
    st->terminated = 1;
  }
}

// linear_system.hpp:67-82 end: chi^2 (kept only on accept), finiteness, max|b|
template <typename FP>
__global__ void k_g_lin_end(GState<FP>* st, Segs<FP> chi, const FP* part_max, unsigned n) {
  if (!st->do_lin) return;
  const FP s = fold_segs(chi);
  const FP gm = block_fold(part_max, n, true);
  if (threadIdx.x != 0) return;
  st->gmax = gm;
  st->finite = (isfinite(s) && !st->bad) ? 1 : 0;
  if (st->accepted) {
    st->chi2 = s;
    st->final_chi2 = static_cast<double>(s);
  }
}

// lambda0 = tau max(D^2 clamped) (linear_system.hpp:94-99), nu = 2
template <typename FP>
__global__ void k_g_init_damping(GState<FP>* st, const FP* part, unsigned n, GCfg c) {
  const FP m = block_fold(part, n, true);
  if (threadIdx.x != 0) return;
  st->lambda = FP(c.tau) * m;
  st->nu = FP(2);
}
#undef GGATE

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
};

inline unsigned nblk(uint64_t n) { return static_cast<unsigned>(std::max<uint64_t>(1, (n + kBlock - 1) / kBlock)); }

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
  using Factor = F;
  static constexpr int kR = F::R;
  uint32_t n = 0;
  std::vector<uint32_t> hidx;
  DVec<uint32_t> idx;
  DVec<typename F::Obs> obs;
  DVec<typename F::Const> cst;
  DVec<FP> J, wr, w, q;
  DVec<uint32_t> off[kMaxSets], item[kMaxSets];
  uint64_t items[kMaxSets] = {0, 0, 0};
  uint64_t part_off = 0;  // this type's slice of the chi^2 partials

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

// per factor type: linearize, accumulate, chi^2, HVP passes (all gated)
template <typename FP, typename F>
struct FactorOps {
  static void lin(cudaStream_t s, const int* on, const Sets<FP>& S, const FSetHost<FP, F>& f, LossCfg l, FP* part) {
    if (!f.n) return;
    k_lin<FP, F><<<nblk(f.n), kBlock, 0, s>>>(on, S, f.dev(), l, part + f.part_off);
    GCK(cudaGetLastError());
  }
  static void chi(cudaStream_t s, const int* on, const Sets<FP>& S, const FSetHost<FP, F>& f, LossCfg l, int cand,
                  FP* part) {
    if (!f.n) return;
    k_chi<FP, F><<<nblk(f.n), kBlock, 0, s>>>(on, S, f.dev(), l, cand, part + f.part_off);
    GCK(cudaGetLastError());
  }
  // many incident items per vertex: one warp per vertex
  static bool wide(const std::vector<VSetHost<FP>*>& sets, const FSetHost<FP, F>& f, int st) {
    return sets[st]->n && f.items[st] >= 16ull * sets[st]->n;
  }
  static void acc(cudaStream_t s, const int* on, const Sets<FP>& S, const std::vector<VSetHost<FP>*>& sets,
                  const FSetHost<FP, F>& f, FP* b, FP* H) {
    for (int st = 0; st < static_cast<int>(sets.size()); ++st) {
      if (!f.off[st].p || !f.n) continue;
      by_dim(sets[st]->dim, [&](auto Dc) {
        constexpr int D = decltype(Dc)::value;
        if (D <= 6 && wide(sets, f, st))
          k_acc_w<FP, F, D><<<nblk(32ull * sets[st]->n), kBlock, 0, s>>>(on, S, f.dev(), st, b, H);
        else
          k_acc<FP, F, D><<<nblk(sets[st]->n), kBlock, 0, s>>>(on, S, f.dev(), st, b, H);
      });
      GCK(cudaGetLastError());
    }
  }
  static void fwd(cudaStream_t s, const int* on, const Sets<FP>& S, const FSetHost<FP, F>& f, const FP* vt) {
    if (!f.n) return;
    if (F::R >= 8)
      k_fwd_w<FP, F><<<nblk(32ull * f.n), kBlock, 0, s>>>(on, S, f.dev(), vt);
    else
      k_fwd<FP, F><<<nblk(f.n), kBlock, 0, s>>>(on, S, f.dev(), vt);
    GCK(cudaGetLastError());
  }
  static void back(cudaStream_t s, const int* on, const Sets<FP>& S, const std::vector<VSetHost<FP>*>& sets,
                   const FSetHost<FP, F>& f, FP* acc) {
    for (int st = 0; st < static_cast<int>(sets.size()); ++st) {
      if (!f.off[st].p || !f.n) continue;
      by_dim(sets[st]->dim, [&](auto Dc) {
        constexpr int D = decltype(Dc)::value;
        if (wide(sets, f, st))
          k_back_w<FP, F, D><<<nblk(32ull * sets[st]->n), kBlock, 0, s>>>(on, S, f.dev(), st, acc);
        else
          k_back<FP, F, D><<<nblk(sets[st]->n), kBlock, 0, s>>>(on, S, f.dev(), st, acc);
      });
      GCK(cudaGetLastError());
    }
  }
};

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
  uint64_t chi_parts = 0;
  m.each([&](auto& f) {
    f.build_csr(m.sets);
    nfactors += f.n;
    residual_dims += static_cast<int64_t>(f.n) * std::remove_reference_t<decltype(f)>::kR;
    f.part_off = chi_parts;
    chi_parts += f.n ? nblk(f.n) : 0;
  });
  uint64_t rz_parts = 0;
  std::vector<uint64_t> rz_off(m.sets.size());
  for (size_t st = 0; st < m.sets.size(); ++st) {
    rz_off[st] = rz_parts;
    rz_parts += nblk(m.sets[st]->n);
  }
  if (m.sets.size() > 4 || sizeof...(Fs) > 4) throw std::invalid_argument("at most 4 vertex sets / factor types");
  const unsigned nbN = nblk(N);
  DVec<FP> b, diag, clamped, Dv, H, M, vt, acc, rhs, xs, r, z, p, ap, part_chi, part_dot, part_max, part_rz, beta;
  for (auto* d : {&b, &diag, &clamped, &Dv, &vt, &acc, &rhs, &xs, &r, &z, &p, &ap}) d->alloc(N);
  H.alloc(hsize);
  M.alloc(hsize);
  part_chi.alloc(chi_parts);
  part_dot.alloc(nbN);
  part_max.alloc(nbN);
  part_rz.alloc(rz_parts);
  beta.alloc(1);
  const int max_it = std::max(0, cfg.max_iterations);
  DVec<gb_iteration_record> drecs;
  drecs.alloc(std::max(1, max_it));
  DVec<GState<FP>> dst;
  dst.alloc(1);
  GState<FP>* st = dst.p;
  const int* on_iter = &st->iter_active;
  const int* on_pcg = &st->pcg_active;
  const int* on_step = &st->step_ok;
  const int* on_acc = &st->accepted;
  const int* on_lin = &st->do_lin;
  const int before = cfg.damping == GB_DAMPING_BEFORE_SCALING ? 1 : 0;
  GCfg gc{max_it, cfg.pcg.max_iterations, cfg.pcg.normalize_rhs, cfg.use_rejection_guard, cfg.refresh_on_reject,
          before, cfg.tolerance, cfg.gradient_tolerance, cfg.lambda_max, cfg.tau, cfg.pcg.tolerance,
          cfg.pcg.rejection_ratio, cfg.clamp_min, cfg.clamp_max};
  Segs<FP> chi_segs{}, rz_segs{};
  {
    int k = 0;
    m.each([&](auto& f) {
      if (f.n) {
        chi_segs.p[k] = part_chi.p + f.part_off;
        chi_segs.n[k] = nblk(f.n);
        ++k;
      }
    });
    chi_segs.count = k;
    for (size_t s2 = 0; s2 < m.sets.size(); ++s2) {
      rz_segs.p[s2] = part_rz.p + rz_off[s2];
      rz_segs.n[s2] = nblk(m.sets[s2]->n);
    }
    rz_segs.count = static_cast<int>(m.sets.size());
  }
  cudaStream_t s;
  GCK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() { cudaStreamDestroy(s); }
  } sg{s};
  auto grid = [](uint64_t n) { return std::max(1u, std::min(nblk(n), 148u * 8u)); };

  auto ops = [&](auto& f) -> FactorOps<FP, typename std::remove_reference_t<decltype(f)>::Factor> { return {}; };

  // LinearSystem::linearize (linear_system.hpp:67-82), gated on do_lin: chi
  // partials, b / H over the CSRs, diag, clamp, D, max|b|, finiteness
  auto enqueue_linearize = [&]() {
    m.each([&](auto& f) { ops(f).lin(s, on_lin, S, f, m.loss, part_chi.p); });
    k_fill<FP><<<grid(N), kBlock, 0, s>>>(on_lin, N, b.p, FP(0));
    k_fill<FP><<<grid(hsize), kBlock, 0, s>>>(on_lin, hsize, H.p, FP(0));
    m.each([&](auto& f) { ops(f).acc(s, on_lin, S, m.sets, f, b.p, H.p); });
    k_fill<FP><<<grid(N), kBlock, 0, s>>>(on_lin, N, diag.p, FP(0));
    for (size_t q = 0; q < m.sets.size(); ++q)
      k_diag<FP><<<nblk(m.sets[q]->n), kBlock, 0, s>>>(on_lin, S, static_cast<int>(q), m.sets[q]->dim, H.p, diag.p);
    k_fill<int><<<1, 32, 0, s>>>(on_lin, 1, &st->bad, 0);
    k_scale<FP><<<nbN, kBlock, 0, s>>>(on_lin, N, b.p, diag.p, cfg.clamp_min, cfg.clamp_max, clamped.p, Dv.p,
                                       part_max.p, &st->bad);
    k_g_lin_end<FP><<<1, kBlock, 0, s>>>(st, chi_segs, part_max.p, nbN);
    GCK(cudaGetLastError());
  };
  auto enqueue_apply_M = [&](FP* part_out) {  // z = M r (per set), r.z partials
    for (size_t q = 0; q < m.sets.size(); ++q)
      by_dim(m.sets[q]->dim, [&](auto Dc) {
        constexpr int Dd = decltype(Dc)::value;
        k_apply<FP, Dd><<<nblk(m.sets[q]->n), kBlock, 0, s>>>(on_pcg, S, static_cast<int>(q), M.p, r.p, z.p,
                                                              part_out + rz_off[q]);
      });
  };
  // One LM iteration (levenberg_marquardt.hpp:149-220) as a fixed kernel
  // sequence with pcg.max_iterations unrolled PCG steps; every kernel is
  // gated by the device state.
  auto enqueue_iteration = [&]() {
    k_g_iter_begin<FP><<<1, 32, 0, s>>>(st, drecs.p, gc);
    // solve_step (linear_system.hpp:185-207): block-Jacobi, PCG (pcg.hpp:34-105), pred, dx
    k_fill<int><<<1, 32, 0, s>>>(on_iter, 1, &st->fallbacks, 0);
    for (size_t q = 0; q < m.sets.size(); ++q)
      by_dim(m.sets[q]->dim, [&](auto Dc) {
        constexpr int Dd = decltype(Dc)::value;
        k_precond<FP, Dd><<<nblk(m.sets[q]->n), kBlock, 0, s>>>(on_iter, S, static_cast<int>(q), H.p, Dv.p, st,
                                                                before, cfg.clamp_min, cfg.clamp_max, M.p,
                                                                &st->fallbacks);
      });
    k_rhs<FP><<<nbN, kBlock, 0, s>>>(on_iter, N, Dv.p, b.p, rhs.p);
    k_dot<FP><<<nbN, kBlock, 0, s>>>(on_iter, N, rhs.p, rhs.p, part_dot.p);
    k_fill<FP><<<grid(N), kBlock, 0, s>>>(on_iter, N, xs.p, FP(0));
    k_g_pcg_begin<FP><<<1, kBlock, 0, s>>>(st, part_dot.p, nbN, gc);
    k_init_r<FP><<<nbN, kBlock, 0, s>>>(on_pcg, N, st, rhs.p, r.p);
    enqueue_apply_M(part_rz.p);
    k_copy<FP><<<grid(N), kBlock, 0, s>>>(on_pcg, N, p.p, z.p);
    k_dot<FP><<<nbN, kBlock, 0, s>>>(on_pcg, N, r.p, r.p, part_dot.p);
    k_g_rho<FP><<<1, kBlock, 0, s>>>(st, rz_segs, part_dot.p, nbN);
    for (int it = 0; it < cfg.pcg.max_iterations; ++it) {
      // A p (LinearSystem::hvp, linear_system.hpp:104-115)
      k_axpy_vt<FP><<<nbN, kBlock, 0, s>>>(on_pcg, N, Dv.p, p.p, vt.p);
      k_fill<FP><<<grid(N), kBlock, 0, s>>>(on_pcg, N, acc.p, FP(0));
      m.each([&](auto& f) {
        ops(f).fwd(s, on_pcg, S, f, vt.p);
        ops(f).back(s, on_pcg, S, m.sets, f, acc.p);
      });
      k_hvp_fin<FP><<<nbN, kBlock, 0, s>>>(on_pcg, N, Dv.p, p.p, acc.p, st, before, ap.p);
      k_dot<FP><<<nbN, kBlock, 0, s>>>(on_pcg, N, p.p, ap.p, part_dot.p);
      k_g_pap<FP><<<1, kBlock, 0, s>>>(st, part_dot.p, nbN);
      k_update_xr<FP><<<nbN, kBlock, 0, s>>>(on_pcg, N, st, p.p, ap.p, xs.p, r.p);
      k_dot<FP><<<nbN, kBlock, 0, s>>>(on_pcg, N, r.p, r.p, part_dot.p);
      k_g_res<FP><<<1, kBlock, 0, s>>>(st, part_dot.p, nbN, gc);
      enqueue_apply_M(part_rz.p);
      k_g_beta<FP><<<1, kBlock, 0, s>>>(st, rz_segs, beta.p);
      k_dir<FP><<<nbN, kBlock, 0, s>>>(on_pcg, N, beta.p, z.p, p.p);
    }
    k_unscale<FP><<<nbN, kBlock, 0, s>>>(on_iter, N, st, xs.p);
    k_pred<FP><<<nbN, kBlock, 0, s>>>(on_iter, N, Dv.p, xs.p, rhs.p, st, before, part_dot.p, &st->badx);
    k_g_step<FP><<<1, kBlock, 0, s>>>(st, drecs.p, part_dot.p, nbN, gc);
    // apply_step + total_error at the candidate (graph.hpp:107-128)
    for (size_t q = 0; q < m.sets.size(); ++q)
      by_dim(m.sets[q]->dim, [&](auto Dc) {
        constexpr int Dd = decltype(Dc)::value;
        k_apply_step<FP, Dd><<<nblk(m.sets[q]->n), kBlock, 0, s>>>(on_step, S, static_cast<int>(q), Dv.p, xs.p);
      });
    m.each([&](auto& f) { ops(f).chi(s, on_step, S, f, m.loss, 1, part_chi.p); });
    k_g_decide<FP><<<1, kBlock, 0, s>>>(st, drecs.p, chi_segs, gc);
    // accept: x <- x_new, then re-linearize (also on reject with refresh_on_reject)
    for (auto* v : m.sets) k_copy<FP><<<grid(v->xn.n), kBlock, 0, s>>>(on_acc, v->xn.n, v->x.p, v->xn.p);
    enqueue_linearize();
    GCK(cudaGetLastError());
  };

  if (rep) std::memset(rep, 0, sizeof(*rep));
  GState<FP> hs{};
  hs.do_lin = 1;
  hs.accepted = 1;  // the initial linearization keeps its chi^2
  GCK(cudaMemcpyAsync(st, &hs, sizeof(hs), cudaMemcpyHostToDevice, s));
  enqueue_linearize();
  GCK(cudaMemcpyAsync(&hs, st, sizeof(hs), cudaMemcpyDeviceToHost, s));
  GCK(cudaStreamSynchronize(s));
  const FP chi2 = hs.chi2;
  if (!std::isfinite(static_cast<double>(chi2)))
    throw std::runtime_error("levenberg_marquardt: non-finite chi^2 at the initial parameters");
  gb_solve_report R{};
  R.initial_chi2 = R.final_chi2 = static_cast<double>(chi2);
  R.free_dims = N;
  R.active_factors = nfactors;
  R.termination = GB_TERM_MAX_ITERATIONS;
  std::vector<gb_iteration_record> its;
  if (N == 0) {
    R.termination = GB_TERM_NO_FREE_PARAMETERS;
  } else if (max_it > 0) {
    k_damp_max<FP><<<nbN, kBlock, 0, s>>>(N, Dv.p, clamped.p, part_max.p);
    hs.it = 0;
    hs.terminated = 0;
    hs.accepted = 0;
    hs.do_lin = 0;
    hs.accepted_steps = 0;
    hs.final_chi2 = static_cast<double>(chi2);
    GCK(cudaMemcpyAsync(st, &hs, sizeof(hs), cudaMemcpyHostToDevice, s));
    k_g_init_damping<FP><<<1, kBlock, 0, s>>>(st, part_max.p, nbN, gc);
    GCK(cudaGetLastError());
    // capture one iteration; replay it, polling the termination flag one
    // iteration behind (the device no-ops iterations after termination)
    cudaGraph_t graph;
    cudaGraphExec_t exec;
    GCK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    enqueue_iteration();
    GCK(cudaStreamEndCapture(s, &graph));
    GCK(cudaGraphInstantiate(&exec, graph, 0));
    GCK(cudaGraphDestroy(graph));
    struct ExecGuard {
      cudaGraphExec_t e;
      ~ExecGuard() { cudaGraphExecDestroy(e); }
    } eg{exec};
    int* hflag = nullptr;
    GCK(cudaHostAlloc(&hflag, sizeof(int) * (max_it + 1), cudaHostAllocDefault));
    struct HostGuard {
      int* p;
      ~HostGuard() { cudaFreeHost(p); }
    } hg{hflag};
    std::vector<cudaEvent_t> ev(max_it + 1);
    for (auto& e : ev) GCK(cudaEventCreate(&e));
    struct EvGuard {
      std::vector<cudaEvent_t>& v;
      ~EvGuard() {
        for (auto e : v) cudaEventDestroy(e);
      }
    } evg{ev};
    GCK(cudaEventRecord(ev[0], s));
    int launched = 0;
    for (int k = 0; k < max_it; ++k) {
      if (k >= 2) {  // iteration k-2 finished: did it terminate?
        GCK(cudaEventSynchronize(ev[k - 1]));
        if (hflag[k - 2]) break;
      }
      GCK(cudaGraphLaunch(exec, s));
      GCK(cudaMemcpyAsync(&hflag[k], &st->terminated, sizeof(int), cudaMemcpyDeviceToHost, s));
      GCK(cudaEventRecord(ev[k + 1], s));
      ++launched;
    }
    GCK(cudaMemcpyAsync(&hs, st, sizeof(hs), cudaMemcpyDeviceToHost, s));
    GCK(cudaStreamSynchronize(s));
    its.resize(hs.it);
    if (hs.it) GCK(cudaMemcpy(its.data(), drecs.p, sizeof(gb_iteration_record) * hs.it, cudaMemcpyDeviceToHost));
    for (int i = 0; i < hs.it && i < launched; ++i) {
      float ms = 0;
      GCK(cudaEventElapsedTime(&ms, ev[i], ev[i + 1]));
      its[i].wall_seconds = 1e-3 * ms;
    }
    R.termination = hs.terminated ? hs.termination : GB_TERM_MAX_ITERATIONS;
    R.accepted_steps = hs.accepted_steps;
    R.final_chi2 = hs.final_chi2;
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
