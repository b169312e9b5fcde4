// Snavely camera model on the device (reference include/gopt/bal/snavely.hpp).
//
// One edge = one observation of point X by camera [w1 w2 w3 t1 t2 t3 f k1 k2].
// The residual follows snavely_project (snavely.hpp:48-61) through the direct
// Rodrigues formula rotate_angle_axis (:18-43); the Jacobians follow the
// analytic chain SnavelyChain (:67-129) built ONCE per edge and shared by the
// 2x9 camera block and the 2x3 point block (the reference builds the chain
// twice, once per slot, adapter.hpp:67-74). Both share the Taylor switch
// kRodriguesTaylorThreshold (:13-14).
#pragma once

#include "common.cuh"

namespace gb {

template <typename FP>
struct taylor_threshold;
template <>
struct taylor_threshold<double> {
  static constexpr double value = 1e-6;
};
template <>
struct taylor_threshold<float> {
  static constexpr float value = 1e-2f;
};

__device__ inline void sin_cos(double x, double* s, double* c) { sincos(x, s, c); }
__device__ inline void sin_cos(float x, float* s, float* c) { sincosf(x, s, c); }

// Rodrigues coefficients shared by the residual and the Jacobian chain:
// a = cos t, s = sin t / t, c = (1 - cos t) / t^2 (snavely.hpp:23-35) and the
// derivative coefficients s1 = (a - s)/t^2, c2 = (s - 2c)/t^2 (:74-90). One
// sqrt, one sincos and two reciprocals per edge (the reference evaluates the
// chain twice per edge and divides each time).
template <typename FP>
struct Rodrigues {
  FP a, s, c;        // residual path (rotate_angle_axis Taylor form)
  FP ja, js, jcc;    // chain path (rodrigues_with_jacobian Taylor form)
  FP s1, c2;
};

template <typename FP>
__device__ inline Rodrigues<FP> rodrigues_coeffs(FP w0, FP w1, FP w2, bool need_chain) {
  Rodrigues<FP> R;
  const FP theta2 = w0 * w0 + w1 * w1 + w2 * w2;
  if (theta2 < taylor_threshold<FP>::value) {
    const FP u = theta2;
    R.a = FP(1) - u * FP(0.5) + u * u * (FP(1) / FP(24));
    R.s = FP(1) - u * (FP(1) / FP(6)) + u * u * (FP(1) / FP(120));
    R.c = FP(0.5) - u * (FP(1) / FP(24)) + u * u * (FP(1) / FP(720));
    if (need_chain) {
      R.ja = FP(1) - u / FP(2) + u * u / FP(24);
      R.js = FP(1) - u / FP(6) + u * u / FP(120);
      R.jcc = FP(0.5) - u / FP(24) + u * u / FP(720);
      R.s1 = -FP(1) / FP(3) + u / FP(30);
      R.c2 = -FP(1) / FP(12) + u / FP(180);
    }
  } else {
    const FP theta = sqrt(theta2);
    FP sn, cs;
    sin_cos(theta, &sn, &cs);
    const FP it2 = FP(1) / theta2;
    R.a = cs;
    R.s = sn / theta;
    R.c = (FP(1) - cs) * it2;
    R.ja = R.a;
    R.js = R.s;
    R.jcc = R.c;
    if (need_chain) {
      R.s1 = (R.a - R.s) * it2;
      R.c2 = (R.s - FP(2) * R.c) * it2;
    }
  }
  return R;
}

// P = R(w) X + t through the direct Rodrigues formula (rotate_angle_axis,
// snavely.hpp:36-42 + :52-54).
template <typename FP>
__device__ inline void rotate_translate(const FP* cam, const FP* X, const Rodrigues<FP>& R, FP* P) {
  const FP w0 = cam[0], w1 = cam[1], w2 = cam[2];
  const FP wx = w1 * X[2] - w2 * X[1];
  const FP wy = w2 * X[0] - w0 * X[2];
  const FP wz = w0 * X[1] - w1 * X[0];
  const FP dot = w0 * X[0] + w1 * X[1] + w2 * X[2];
  P[0] = R.a * X[0] + R.s * wx + R.c * dot * w0 + cam[3];
  P[1] = R.a * X[1] + R.s * wy + R.c * dot * w1 + cam[4];
  P[2] = R.a * X[2] + R.s * wz + R.c * dot * w2 + cam[5];
}

// Residual r = predicted - observed (adapter.hpp:58-65, snavely.hpp:48-61).
template <typename FP>
__device__ inline void snavely_residual(const FP* cam, const FP* X, FP o0, FP o1, FP* r) {
  const Rodrigues<FP> R = rodrigues_coeffs<FP>(cam[0], cam[1], cam[2], false);
  FP P[3];
  rotate_translate(cam, X, R, P);
  const FP iz = FP(1) / P[2];
  const FP xp = -P[0] * iz, yp = -P[1] * iz;
  const FP n = xp * xp + yp * yp;
  const FP d = FP(1) + n * (cam[7] + n * cam[8]);
  r[0] = cam[6] * d * xp - o0;
  r[1] = cam[6] * d * yp - o1;
}

// Residual and both Jacobian blocks from ONE chain (SnavelyChain,
// snavely.hpp:103-153): jc = d pred / d camera (2x9 row-major),
// jp = d pred / d point (2x3 row-major). r may be null.
// R = a I + s [w]x + c w w^T (rodrigues_with_jacobian, snavely.hpp:67-101),
// explicitly rounded: the factored J store rebuilds the point block from this
// per-camera matrix, so linearize and the HVP must produce identical bits.
template <typename FP>
__device__ inline void rotation_matrix(const Rodrigues<FP>& Ro, FP w0, FP w1, FP w2, FP* R) {
  const FP a = Ro.ja, s = Ro.js, c = Ro.jcc;
  const FP c0 = mul_rn(c, w0), c1 = mul_rn(c, w1), c2 = mul_rn(c, w2);
  R[0] = fma_rn(c0, w0, a);
  R[1] = fma_rn(c0, w1, -mul_rn(s, w2));
  R[2] = fma_rn(c0, w2, mul_rn(s, w1));
  R[3] = fma_rn(c1, w0, mul_rn(s, w2));
  R[4] = fma_rn(c1, w1, a);
  R[5] = fma_rn(c1, w2, -mul_rn(s, w0));
  R[6] = fma_rn(c2, w0, -mul_rn(s, w1));
  R[7] = fma_rn(c2, w1, mul_rn(s, w0));
  R[8] = fma_rn(c2, w2, a);
}

// Point block jp = du/dP . R (snavely.hpp:150-153), 2x3 row-major.
template <typename FP>
__device__ inline void point_block(const FP* U, const FP* R, FP* jp) {
#pragma unroll
  for (int rr = 0; rr < 2; ++rr)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      jp[3 * rr + j] = fma_rn(U[3 * rr + 2], R[6 + j], fma_rn(U[3 * rr + 1], R[3 + j], mul_rn(U[3 * rr], R[j])));
}

// Intrinsics columns of the camera block: [d p | f n p | f n^2 p]
// (snavely.hpp:122-128).
template <typename FP>
__device__ inline void intrinsic_cols(FP dist, FP n, FP p0, FP p1, FP f, FP* jc) {
  const FP fn = mul_rn(f, n), fnn = mul_rn(fn, n);
  jc[6] = mul_rn(dist, p0);
  jc[15] = mul_rn(dist, p1);
  jc[7] = mul_rn(fn, p0);
  jc[16] = mul_rn(fn, p1);
  jc[8] = mul_rn(fnn, p0);
  jc[17] = mul_rn(fnn, p1);
}

// Per-camera record of the factored J store: R (9) and f.
template <typename FP>
__device__ inline void camera_factor(const FP* cam, FP* rf) {
  const Rodrigues<FP> Ro = rodrigues_coeffs<FP>(cam[0], cam[1], cam[2], true);
  rotation_matrix<FP>(Ro, cam[0], cam[1], cam[2], rf);
  rf[9] = cam[6];
}

// ---- per-camera precomputation ---------------------------------------------
// Everything of the chain that depends on the camera alone (one sqrt, one
// sincos, two reciprocals and the rotation matrix) is computed once per camera
// per linearization / candidate evaluation (k_cam_pre) instead of once per
// edge; the per-edge functions below read it. Record: [a s c ja js jcc s1 c2 |
// R (9) | pad] (kCamPre values).
constexpr int kCamPre = 18;

template <typename FP>
__device__ inline void camera_pre(const FP* cam, FP* pre) {
  const Rodrigues<FP> Ro = rodrigues_coeffs<FP>(cam[0], cam[1], cam[2], true);
  pre[0] = Ro.a;
  pre[1] = Ro.s;
  pre[2] = Ro.c;
  pre[3] = Ro.ja;
  pre[4] = Ro.js;
  pre[5] = Ro.jcc;
  pre[6] = Ro.s1;
  pre[7] = Ro.c2;
  rotation_matrix<FP>(Ro, cam[0], cam[1], cam[2], pre + 8);
  pre[17] = FP(0);
}

template <typename FP>
__device__ inline Rodrigues<FP> rodrigues_from_pre(const FP* pre) {
  Rodrigues<FP> R;
  R.a = pre[0];
  R.s = pre[1];
  R.c = pre[2];
  R.ja = pre[3];
  R.js = pre[4];
  R.jcc = pre[5];
  R.s1 = pre[6];
  R.c2 = pre[7];
  return R;
}

// snavely_residual with the camera's precomputed record
template <typename FP>
__device__ inline void snavely_residual_pre(const FP* cam, const FP* pre, const FP* X, FP o0, FP o1, FP* r) {
  const Rodrigues<FP> R = rodrigues_from_pre(pre);
  FP P[3];
  rotate_translate(cam, X, R, P);
  const FP iz = FP(1) / P[2];
  const FP xp = -P[0] * iz, yp = -P[1] * iz;
  const FP n = xp * xp + yp * yp;
  const FP d = FP(1) + n * (cam[7] + n * cam[8]);
  r[0] = cam[6] * d * xp - o0;
  r[1] = cam[6] * d * yp - o1;
}

template <typename FP>
__device__ inline void snavely_linearize(const FP* cam, const FP* X, FP o0, FP o1, FP* r, FP* jc, FP* jp,
                                         FP* fac = nullptr, const FP* pre = nullptr) {
  const FP w0 = cam[0], w1 = cam[1], w2 = cam[2];
  const FP x0 = X[0], x1 = X[1], x2 = X[2];
  const Rodrigues<FP> Ro = pre ? rodrigues_from_pre(pre) : rodrigues_coeffs<FP>(w0, w1, w2, true);
  FP P[3];
  rotate_translate(cam, X, Ro, P);
  const FP s = Ro.js, c = Ro.jcc, s1 = Ro.s1, c2 = Ro.c2;
  FP R[9];
  if (pre) {
#pragma unroll
    for (int k = 0; k < 9; ++k) R[k] = pre[8 + k];
  } else {
    rotation_matrix<FP>(Ro, w0, w1, w2, R);
  }
  // dy/dw = -s x w^T + s1 (w x x) w^T - s [x]x + c2 (w.x) w w^T + c (w x^T + (w.x) I)
  const FP cr[3] = {w1 * x2 - w2 * x1, w2 * x0 - w0 * x2, w0 * x1 - w1 * x0};
  const FP dt = w0 * x0 + w1 * x1 + w2 * x2;
  const FP w[3] = {w0, w1, w2};
  const FP x[3] = {x0, x1, x2};
  const FP skx[9] = {FP(0), -x2, x1, x2, FP(0), -x0, -x1, x0, FP(0)};
  FP Dw[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      Dw[3 * i + j] = -s * x[i] * w[j] + s1 * cr[i] * w[j] - s * skx[3 * i + j] + c2 * dt * w[i] * w[j] +
                      c * (w[i] * x[j] + (i == j ? dt : FP(0)));
  const FP iz = FP(1) / P[2];
  const FP p0 = -P[0] * iz, p1 = -P[1] * iz;
  const FP n = p0 * p0 + p1 * p1;
  const FP f = cam[6], k1 = cam[7], k2 = cam[8];
  const FP dist = FP(1) + n * (k1 + n * k2);
  if (r) {
    r[0] = f * dist * p0 - o0;
    r[1] = f * dist * p1 - o1;
  }
  // du/dp = f (dist I + 2 (k1 + 2 k2 n) p p^T); dp/dP = [[-iz,0,P0 iz^2],[0,-iz,P1 iz^2]]
  const FP g = FP(2) * (k1 + FP(2) * k2 * n);
  const FP A00 = f * (dist + g * p0 * p0), A01 = f * (g * p0 * p1);
  const FP A10 = f * (g * p1 * p0), A11 = f * (dist + g * p1 * p1);
  const FP iz2 = iz * iz;
  const FP B02 = P[0] * iz2, B12 = P[1] * iz2;
  FP U[6];  // du/dP 2x3
  U[0] = -A00 * iz;
  U[1] = -A01 * iz;
  U[2] = A00 * B02 + A01 * B12;
  U[3] = -A10 * iz;
  U[4] = -A11 * iz;
  U[5] = A10 * B02 + A11 * B12;
#pragma unroll
  for (int rr = 0; rr < 2; ++rr) {
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      jc[9 * rr + j] = U[3 * rr] * Dw[j] + U[3 * rr + 1] * Dw[3 + j] + U[3 * rr + 2] * Dw[6 + j];
      jc[9 * rr + 3 + j] = U[3 * rr + j];
    }
  }
  point_block<FP>(U, R, jp);
  intrinsic_cols<FP>(dist, n, p0, p1, f, jc);
  if (fac) {  // factored store: U (6), dist, n, p0, p1
#pragma unroll
    for (int k = 0; k < 6; ++k) fac[k] = U[k];
    fac[6] = dist;
    fac[7] = n;
    fac[8] = p0;
    fac[9] = p1;
  }
}

template <typename FP>
__device__ inline void snavely_jacobians(const FP* cam, const FP* X, FP* jc, FP* jp) {
  snavely_linearize<FP>(cam, X, FP(0), FP(0), nullptr, jc, jp);
}

// ---- Auto differentiation (DifferentiationMode::Auto) ----------------------
// Forward-mode dual numbers with one infinitesimal (dual.hpp:13-99) and the
// residual evaluated generically (snavely_project + rotate_angle_axis,
// snavely.hpp:18-61): one pass per Jacobian column, the residual recomputed
// per column exactly like FactorDescriptor::jacobian_auto_slot
// (factor_descriptor.hpp:610-624).
template <typename T>
struct Dual {
  T v, d;
};
template <typename T>
__device__ inline Dual<T> operator+(Dual<T> a, Dual<T> b) { return {a.v + b.v, a.d + b.d}; }
template <typename T>
__device__ inline Dual<T> operator-(Dual<T> a, Dual<T> b) { return {a.v - b.v, a.d - b.d}; }
template <typename T>
__device__ inline Dual<T> operator*(Dual<T> a, Dual<T> b) { return {a.v * b.v, a.v * b.d + a.d * b.v}; }
template <typename T>
__device__ inline Dual<T> operator/(Dual<T> a, Dual<T> b) {
  const T inv = T(1) / b.v;
  return {a.v * inv, (a.d - a.v * inv * b.d) * inv};
}
template <typename T>
__device__ inline Dual<T> operator-(Dual<T> a) { return {-a.v, -a.d}; }
template <typename T>
__device__ inline Dual<T> operator+(Dual<T> a, T b) { return {a.v + b, a.d}; }
template <typename T>
__device__ inline Dual<T> operator+(T a, Dual<T> b) { return {a + b.v, b.d}; }
template <typename T>
__device__ inline Dual<T> operator-(Dual<T> a, T b) { return {a.v - b, a.d}; }
template <typename T>
__device__ inline Dual<T> operator-(T a, Dual<T> b) { return {a - b.v, -b.d}; }
template <typename T>
__device__ inline Dual<T> operator*(Dual<T> a, T b) { return {a.v * b, a.d * b}; }
template <typename T>
__device__ inline Dual<T> operator*(T a, Dual<T> b) { return {a * b.v, a * b.d}; }
template <typename T>
__device__ inline Dual<T> dsqrt(Dual<T> a) {
  const T s = sqrt(a.v);
  return {s, a.d / (T(2) * s)};
}
template <typename T>
__device__ inline void dsincos(Dual<T> a, Dual<T>* sn, Dual<T>* cs) {
  T s, c;
  sin_cos(a.v, &s, &c);
  *sn = {s, c * a.d};
  *cs = {c, -s * a.d};
}

// Rodrigues coefficients a, s, c of rotate_angle_axis (snavely.hpp:18-35) on duals
template <typename FP>
__device__ inline void dual_rot_coeffs(const Dual<FP>* omega, Dual<FP>* a, Dual<FP>* s, Dual<FP>* c) {
  using D = Dual<FP>;
  const D theta2 = omega[0] * omega[0] + omega[1] * omega[1] + omega[2] * omega[2];
  if (theta2.v < taylor_threshold<FP>::value) {
    const D u = theta2;
    *a = FP(1) - u * FP(0.5) + u * u * (FP(1) / FP(24));
    *s = FP(1) - u * (FP(1) / FP(6)) + u * u * (FP(1) / FP(120));
    *c = FP(0.5) - u * (FP(1) / FP(24)) + u * u * (FP(1) / FP(720));
  } else {
    const D theta = dsqrt(theta2);
    D sn, cs;
    dsincos(theta, &sn, &cs);
    *a = cs;
    *s = sn / theta;
    *c = (FP(1) - *a) / theta2;
  }
}

// rot (optional): the coefficients of a pass whose rotation is not seeded
// (their derivative parts are 0), computed once per edge
template <typename FP>
__device__ inline void snavely_project_dual(const Dual<FP>* camera, const Dual<FP>* X, Dual<FP>* predicted,
                                            const Dual<FP>* rot = nullptr) {
  using D = Dual<FP>;
  const D* omega = camera;
  D a, s, c;
  if (rot) {
    a = rot[0];
    s = rot[1];
    c = rot[2];
  } else {
    dual_rot_coeffs<FP>(omega, &a, &s, &c);
  }
  const D wx = omega[1] * X[2] - omega[2] * X[1];
  const D wy = omega[2] * X[0] - omega[0] * X[2];
  const D wz = omega[0] * X[1] - omega[1] * X[0];
  const D dot = omega[0] * X[0] + omega[1] * X[1] + omega[2] * X[2];
  D p0 = a * X[0] + s * wx + c * dot * omega[0];
  D p1 = a * X[1] + s * wy + c * dot * omega[1];
  D p2 = a * X[2] + s * wz + c * dot * omega[2];
  p0 = p0 + camera[3];
  p1 = p1 + camera[4];
  p2 = p2 + camera[5];
  const D xp = -p0 / p2;
  const D yp = -p1 / p2;
  const D n = xp * xp + yp * yp;
  const D distortion = FP(1) + n * (camera[7] + n * camera[8]);
  predicted[0] = camera[6] * distortion * xp;
  predicted[1] = camera[6] * distortion * yp;
}

// jc (2x9) and jp (2x3) by 12 dual passes
template <typename FP>
__device__ inline void snavely_jacobians_auto(const FP* cam, const FP* X, FP* jc, FP* jp) {
  // passes 3..11 seed t, f, k1, k2 or X: the rotation coefficients are those
  // of an unseeded omega, computed once (sqrt/sincos/divisions not repeated)
  Dual<FP> rot[3];
  {
    Dual<FP> w0[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) w0[i] = {cam[i], FP(0)};
    dual_rot_coeffs<FP>(w0, &rot[0], &rot[1], &rot[2]);
  }
#pragma unroll 1
  for (int k = 0; k < 12; ++k) {
    Dual<FP> c[9], x[3], pred[2];
#pragma unroll
    for (int i = 0; i < 9; ++i) c[i] = {cam[i], i == k ? FP(1) : FP(0)};
#pragma unroll
    for (int i = 0; i < 3; ++i) x[i] = {X[i], 9 + i == k ? FP(1) : FP(0)};
    snavely_project_dual<FP>(c, x, pred, k < 3 ? nullptr : rot);
    if (k < 9) {
      jc[k] = pred[0].d;
      jc[9 + k] = pred[1].d;
    } else {
      jp[k - 9] = pred[0].d;
      jp[3 + k - 9] = pred[1].d;
    }
  }
}

// Robust loss (loss.hpp:25-40): value rho(s) and IRLS weight rho'(s).
template <typename FP>
__device__ inline FP loss_value(int kind, FP delta, FP s) {
  if (kind == 0) return s;
  const FP d2 = delta * delta;
  if (s <= d2) return s;
  return FP(2) * delta * sqrt(s) - d2;
}
template <typename FP>
__device__ inline FP loss_weight(int kind, FP delta, FP s) {
  if (kind == 0) return FP(1);
  const FP d2 = delta * delta;
  if (s <= d2) return FP(1);
  return delta / sqrt(s);
}

}  // namespace gb
