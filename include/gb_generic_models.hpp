/* Host-device factor and vertex models for the generic n-ary factor path
 * (SURVEY.md §8 f-4): the same source is compiled by g++ into the reference's
 * own generic CPU engine (gopt::FactorDescriptor / VertexDescriptor traits,
 * factor_descriptor.hpp:139-151, vertex_descriptor.hpp:50-56; driver
 * oracle/ref_generic.cpp) and by nvcc into the device engine
 * (paper_2509_26581_b200/csrc/generic.cu), so both solve the identical model
 * and the device path's parity is pinned against the reference engine.
 *
 * A residual is a template over the scalar T (FP, or a forward-mode dual
 * number: gopt::Dual on the host, gbg::Dual on the device) and may use + - *
 * /, sqrt, sin, cos and value_of(x) (branch on magnitudes), found by ADL.
 *
 * Models:
 *   circle  the reference's toy (toy/circle.hpp:30-55): 2-D points,
 *           e = x^2 + y^2 - r^2.
 *   vi      an EuRoC-shaped global visual-inertial BA: body poses
 *           [w (angle-axis, body->world) | p], velocity + gyro/accel biases
 *           [v | bg | ba], landmarks X; stereo reprojection factors
 *           (pose, landmark; 3 residuals) and IMU preintegration factors
 *           (pose_i, vb_i, pose_j, vb_j; 15 residuals: position, velocity,
 *           rotation, bias random walks). No reference counterpart exists
 *           (SPEC.md:14); parity is pinned by running these same traits in
 *           the reference's generic engine. */
#pragma once

#include <cmath>
#include <cstdint>

#ifdef __CUDACC__
#define GB_HD __host__ __device__
#else
#define GB_HD
#endif

namespace gbm {

template <typename T>
GB_HD inline T value_of(T x) {
  return x;
}

// ------------------------------------------------------------------ circle
struct CircleObs {
  double radius;
};

template <typename T>
GB_HD inline void circle_residual(const T* point, const CircleObs& o, T* e) {
  const T x = point[0], y = point[1];
  e[0] = x * x + y * y - T(o.radius) * T(o.radius);
}

// ---------------------------------------------------------------------- vi
// R(w) = a I + s [w]x + c w w^T, Taylor form below 1e-8 (rotation matrix of an
// angle-axis vector, snavely.hpp:18-43's coefficients).
template <typename T>
GB_HD inline void rotation(const T* w, T* R) {
  using std::cos;
  using std::sin;
  using std::sqrt;
  const T t2 = w[0] * w[0] + w[1] * w[1] + w[2] * w[2];
  T a, s, c;
  if (value_of(t2) < 1e-8) {
    a = T(1) - t2 * T(0.5);
    s = T(1) - t2 * T(1.0 / 6.0);
    c = T(0.5) - t2 * T(1.0 / 24.0);
  } else {
    const T th = sqrt(t2);
    a = cos(th);
    s = sin(th) / th;
    c = (T(1) - a) / t2;
  }
  R[0] = a + c * w[0] * w[0];
  R[1] = -s * w[2] + c * w[0] * w[1];
  R[2] = s * w[1] + c * w[0] * w[2];
  R[3] = s * w[2] + c * w[1] * w[0];
  R[4] = a + c * w[1] * w[1];
  R[5] = -s * w[0] + c * w[1] * w[2];
  R[6] = -s * w[1] + c * w[2] * w[0];
  R[7] = s * w[0] + c * w[2] * w[1];
  R[8] = a + c * w[2] * w[2];
}

struct StereoObs {
  double uL, vL, uR;
};
struct StereoCam {
  double fx, fy, cx, cy, baseline;
};

// camera = body; P = R(w)^T (X - p); left / right pinhole projections
template <typename T>
GB_HD inline void stereo_residual(const T* pose, const T* X, const StereoObs& o, const StereoCam& k, T* e) {
  T R[9];
  rotation(pose, R);
  const T d0 = X[0] - pose[3], d1 = X[1] - pose[4], d2 = X[2] - pose[5];
  const T P0 = R[0] * d0 + R[3] * d1 + R[6] * d2;
  const T P1 = R[1] * d0 + R[4] * d1 + R[7] * d2;
  const T P2 = R[2] * d0 + R[5] * d1 + R[8] * d2;
  const T iz = T(1) / P2;
  e[0] = T(k.fx) * P0 * iz + T(k.cx) - T(o.uL);
  e[1] = T(k.fy) * P1 * iz + T(k.cy) - T(o.vL);
  e[2] = T(k.fx) * (P0 - T(k.baseline)) * iz + T(k.cx) - T(o.uR);
}

struct ImuObs {
  double dp[3], dv[3], dR[9];  // preintegrated position / velocity / rotation (row-major)
  double dt;
};
struct ImuConst {
  double g[3];  // gravity in the world frame
};

template <typename T>
GB_HD inline void imu_residual(const T* pi, const T* vbi, const T* pj, const T* vbj, const ImuObs& o,
                               const ImuConst& k, T* e) {
  T Ri[9], Rj[9];
  rotation(pi, Ri);
  rotation(pj, Rj);
  const T dt = T(o.dt), hdt2 = T(0.5 * o.dt * o.dt);
  T a[3], b[3];
  for (int q = 0; q < 3; ++q) {
    a[q] = pj[3 + q] - pi[3 + q] - vbi[q] * dt - T(k.g[q]) * hdt2;
    b[q] = vbj[q] - vbi[q] - T(k.g[q]) * dt;
  }
  for (int q = 0; q < 3; ++q) {  // R_i^T a - dp, R_i^T b - dv
    e[q] = Ri[q] * a[0] + Ri[3 + q] * a[1] + Ri[6 + q] * a[2] - T(o.dp[q]);
    e[3 + q] = Ri[q] * b[0] + Ri[3 + q] * b[1] + Ri[6 + q] * b[2] - T(o.dv[q]);
  }
  // E = dR^T R_i^T R_j; rotation error = vee(E - E^T) / 2
  T M[9], E[9];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) M[3 * r + c] = Ri[r] * Rj[c] + Ri[3 + r] * Rj[3 + c] + Ri[6 + r] * Rj[6 + c];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c)
      E[3 * r + c] = T(o.dR[r]) * M[c] + T(o.dR[3 + r]) * M[3 + c] + T(o.dR[6 + r]) * M[6 + c];
  e[6] = T(0.5) * (E[7] - E[5]);
  e[7] = T(0.5) * (E[2] - E[6]);
  e[8] = T(0.5) * (E[3] - E[1]);
  for (int q = 0; q < 6; ++q) e[9 + q] = vbj[3 + q] - vbi[3 + q];
}

}  // namespace gbm
