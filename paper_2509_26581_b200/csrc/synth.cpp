// Synthetic BAL-shaped bundle-adjustment problems (bench and test input).
//
// Semantics follow the reference's own generator, tests/synthetic_bal.hpp:16-113:
// a ring of cameras (radius 10, z ~ U[-1,1]) looking outward so a point cloud
// in [-2,2]^3 sits at negative depth, f=800 k1=-0.05 k2=0.005 ground truth,
// 1 px Gaussian pixel noise, and a perturbed initial estimate (points 0.08,
// rotation 0.008 rad, translation 0.05, f*(1+0.004 N), k1+1e-3 N, k2+1e-4 N).
// Differences, all needed to hit an exact published (cameras, points,
// observations) shape, are documented in DESIGN.md §Inputs:
//   * per-point degree floor(E/np), the first E mod np points get one more;
//   * camera stride grows with the camera count (the reference's stride 3
//     leaves depth ill-conditioned at 13,682 cameras);
//   * Gaussian draws use Box–Muller over mt19937_64 (the reference's own
//     portable NormalSampler, toy/circle.hpp:74-99) instead of libstdc++'s
//     std::normal_distribution, so outputs do not depend on the C++ library;
//   * optional Zipf(s) law for each point's first camera (skewed camera
//     degrees, load-balance stress).
// Edges are written point-grouped, as in BAL files.

#include <cmath>
#include <cstdint>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "gb_bal.h"

namespace {

class Normal {
 public:
  explicit Normal(std::mt19937_64& r) : rng_(r) {}
  double uniform() { return (static_cast<double>(rng_() >> 11) + 1.0) * 0x1.0p-53; }  // (0,1]
  double next() {
    if (have_) {
      have_ = false;
      return spare_;
    }
    const double u1 = uniform(), u2 = uniform();
    const double mag = std::sqrt(-2.0 * std::log(u1));
    spare_ = mag * std::sin(2.0 * M_PI * u2);
    have_ = true;
    return mag * std::cos(2.0 * M_PI * u2);
  }

 private:
  std::mt19937_64& rng_;
  double spare_ = 0;
  bool have_ = false;
};

struct Cam {
  double R[9];  // row-major
  double t[3];
};

// Rotation matrix -> angle-axis via a unit quaternion (Shepperd), robust for
// angles up to pi (the outward-looking ring spans every heading).
void log_map(const double* R, double* w) {
  const double tr = R[0] + R[4] + R[8];
  double q[4];  // w x y z
  if (tr > 0) {
    const double s = std::sqrt(tr + 1.0) * 2;
    q[0] = 0.25 * s;
    q[1] = (R[7] - R[5]) / s;
    q[2] = (R[2] - R[6]) / s;
    q[3] = (R[3] - R[1]) / s;
  } else if (R[0] > R[4] && R[0] > R[8]) {
    const double s = std::sqrt(1.0 + R[0] - R[4] - R[8]) * 2;
    q[0] = (R[7] - R[5]) / s;
    q[1] = 0.25 * s;
    q[2] = (R[1] + R[3]) / s;
    q[3] = (R[2] + R[6]) / s;
  } else if (R[4] > R[8]) {
    const double s = std::sqrt(1.0 + R[4] - R[0] - R[8]) * 2;
    q[0] = (R[2] - R[6]) / s;
    q[1] = (R[1] + R[3]) / s;
    q[2] = 0.25 * s;
    q[3] = (R[5] + R[7]) / s;
  } else {
    const double s = std::sqrt(1.0 + R[8] - R[0] - R[4]) * 2;
    q[0] = (R[3] - R[1]) / s;
    q[1] = (R[2] + R[6]) / s;
    q[2] = (R[5] + R[7]) / s;
    q[3] = 0.25 * s;
  }
  if (q[0] < 0)
    for (double& v : q) v = -v;
  const double vn = std::sqrt(q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
  if (vn < 1e-300) {
    w[0] = w[1] = w[2] = 0;
    return;
  }
  const double angle = 2.0 * std::atan2(vn, q[0]);
  for (int k = 0; k < 3; ++k) w[k] = angle * q[k + 1] / vn;
}

void project(const Cam& c, const double* x, double f, double k1, double k2, double* uv) {
  double P[3];
  for (int i = 0; i < 3; ++i) P[i] = c.R[3 * i] * x[0] + c.R[3 * i + 1] * x[1] + c.R[3 * i + 2] * x[2] + c.t[i];
  const double px = -P[0] / P[2], py = -P[1] / P[2];
  const double n = px * px + py * py;
  const double d = 1 + n * (k1 + n * k2);
  uv[0] = f * d * px;
  uv[1] = f * d * py;
}

}  // namespace

extern "C" int gb_synthetic_bal(uint64_t nc, uint64_t np, uint64_t ne, uint64_t seed,
                                uint64_t stride, double zipf_s, uint32_t* cam_out,
                                uint32_t* pt_out, double* obs_out, double* cams_out,
                                double* pts_out) {
  if (nc == 0 || np == 0 || ne < np) return GB_ERR_INVALID_ARGUMENT;
  const uint64_t base = ne / np, extra = ne % np;
  const uint64_t dmax = base + (extra ? 1 : 0);
  if (dmax > nc) return GB_ERR_INVALID_ARGUMENT;  // a point cannot see a camera twice
  if (stride == 0) stride = nc / (dmax + 1) > 0 ? nc / (dmax + 1) : 1;
  if ((dmax - 1) * stride >= nc) stride = 1;  // keep the cameras of one point distinct

  std::mt19937_64 rng(seed);
  Normal gauss(rng);

  std::vector<double> gt(3 * np);
  for (uint64_t p = 0; p < np; ++p)
    for (int k = 0; k < 3; ++k) gt[3 * p + k] = 4 * gauss.uniform() - 2;

  std::vector<Cam> cams(nc);
  const double f0 = 800.0, k10 = -0.05, k20 = 0.005;
  for (uint64_t i = 0; i < nc; ++i) {
    const double angle = 2 * M_PI * static_cast<double>(i) / static_cast<double>(nc);
    const double center[3] = {10 * std::cos(angle), 10 * std::sin(angle), 2 * gauss.uniform() - 1};
    const double cn = std::sqrt(center[0] * center[0] + center[1] * center[1] + center[2] * center[2]);
    const double zc[3] = {center[0] / cn, center[1] / cn, center[2] / cn};
    double xc[3] = {-zc[1], zc[0], 0.0};  // UnitZ x zc
    const double xn = std::sqrt(xc[0] * xc[0] + xc[1] * xc[1]);
    xc[0] /= xn;
    xc[1] /= xn;
    const double yc[3] = {zc[1] * xc[2] - zc[2] * xc[1], zc[2] * xc[0] - zc[0] * xc[2],
                          zc[0] * xc[1] - zc[1] * xc[0]};
    Cam& c = cams[i];
    for (int k = 0; k < 3; ++k) {
      c.R[k] = xc[k];
      c.R[3 + k] = yc[k];
      c.R[6 + k] = zc[k];
    }
    for (int r = 0; r < 3; ++r)
      c.t[r] = -(c.R[3 * r] * center[0] + c.R[3 * r + 1] * center[1] + c.R[3 * r + 2] * center[2]);
  }

  std::vector<double> zipf_cdf;
  if (zipf_s > 0) {
    zipf_cdf.resize(nc);
    double acc = 0;
    for (uint64_t k = 0; k < nc; ++k) {
      acc += 1.0 / std::pow(static_cast<double>(k + 1), zipf_s);
      zipf_cdf[k] = acc;
    }
    for (double& v : zipf_cdf) v /= acc;
  }

  uint64_t e = 0;
  for (uint64_t p = 0; p < np; ++p) {
    uint64_t start;
    if (zipf_s > 0) {
      const double u = gauss.uniform();
      uint64_t lo = 0, hi = nc - 1;
      while (lo < hi) {
        const uint64_t mid = (lo + hi) / 2;
        if (zipf_cdf[mid] < u) lo = mid + 1; else hi = mid;
      }
      start = lo;
    } else {
      start = rng() % nc;
    }
    const uint64_t deg = base + (p < extra ? 1 : 0);
    for (uint64_t k = 0; k < deg; ++k) {
      const uint64_t ci = (start + k * stride + 1) % nc;
      double uv[2];
      project(cams[ci], &gt[3 * p], f0, k10, k20, uv);
      cam_out[e] = static_cast<uint32_t>(ci);
      pt_out[e] = static_cast<uint32_t>(p);
      obs_out[2 * e] = uv[0] + gauss.next();
      obs_out[2 * e + 1] = uv[1] + gauss.next();
      ++e;
    }
  }

  for (uint64_t i = 0; i < nc; ++i) {
    double* o = cams_out + 9 * i;
    log_map(cams[i].R, o);
    for (int k = 0; k < 3; ++k) o[3 + k] = cams[i].t[k];
    o[6] = f0;
    o[7] = k10;
    o[8] = k20;
    for (int k = 0; k < 3; ++k) o[k] += 0.008 * gauss.next();
    for (int k = 3; k < 6; ++k) o[k] += 0.05 * gauss.next();
    o[6] *= 1.0 + 0.004 * gauss.next();
    o[7] += 1e-3 * gauss.next();
    o[8] += 1e-4 * gauss.next();
  }
  for (uint64_t p = 0; p < np; ++p)
    for (int k = 0; k < 3; ++k) pts_out[3 * p + k] = gt[3 * p + k] + 0.08 * gauss.next();
  return GB_OK;
}
