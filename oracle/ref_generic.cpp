// TEST INFRASTRUCTURE ONLY: the reference's generic CPU engine
// (gopt::VertexDescriptor / FactorDescriptor / Graph / levenberg_marquardt,
// unmodified headers from /root/reference) solving the host-device models of
// include/gb_generic_models.hpp, behind a C ABI. The device engine
// (paper_2509_26581_b200/csrc/generic.cu) exposes the same entry points, so a
// test runs both on identical inputs (the VI config has no
// reference counterpart; its parity is pinned by the reference's own engine
// running the same traits).
//
// Vertex traits follow vertex_descriptor.hpp:50-56 (additive update), factor
// traits factor_descriptor.hpp:139-151 (templated residual, Auto Jacobians via
// gopt::Dual, factor_descriptor.hpp:610-624).
#include <array>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "gb_bal.h"
#include "gb_generic_models.hpp"
#include "gopt/dual.hpp"
#include "gopt/graph.hpp"
#include "gopt/levenberg_marquardt.hpp"

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    g_err.clear();
    return GB_OK;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return GB_ERR_INVALID_ARGUMENT;
  } catch (const std::exception& e) {
    g_err = e.what();
    return GB_ERR_RUNTIME;
  }
}

gopt::LMConfig to_lm(const gb_lm_config& c) {
  gopt::LMConfig lm;
  lm.max_iterations = c.max_iterations;
  lm.tolerance = c.tolerance;
  lm.level = c.level;
  lm.tau = c.tau;
  lm.pcg.max_iterations = c.pcg.max_iterations;
  lm.pcg.tolerance = c.pcg.tolerance;
  lm.pcg.rejection_ratio = c.pcg.rejection_ratio;
  lm.pcg.normalize_rhs = c.pcg.normalize_rhs != 0;
  lm.linear.clamp_min = c.clamp_min;
  lm.linear.clamp_max = c.clamp_max;
  lm.linear.damping = c.damping == GB_DAMPING_BEFORE_SCALING ? gopt::DampingPlacement::before_scaling
                                                             : gopt::DampingPlacement::after_scaling;
  lm.use_rejection_guard = c.use_rejection_guard != 0;
  lm.refresh_on_reject = c.refresh_on_reject != 0;
  lm.lambda_max = c.lambda_max;
  lm.gradient_tolerance = c.gradient_tolerance;
  return lm;
}

void fill(const gopt::SolveReport& r, gb_solve_report* rep, gb_iteration_record* recs, int max_recs) {
  if (rep) {
    std::memset(rep, 0, sizeof(*rep));
    rep->initial_chi2 = r.initial_chi2;
    rep->final_chi2 = r.final_chi2;
    rep->accepted_steps = r.accepted_steps;
    rep->termination = static_cast<int>(r.termination);
    rep->total_seconds = r.total_seconds;
    rep->free_dims = r.free_dims;
    rep->residual_dims = r.residual_dims;
    rep->active_factors = r.active_factors;
    rep->iterations_run = static_cast<std::int32_t>(r.iterations.size());
  }
  if (recs) {
    const int n = std::min<int>(max_recs, static_cast<int>(r.iterations.size()));
    for (int i = 0; i < n; ++i) {
      const auto& it = r.iterations[i];
      recs[i] = {it.iteration,       it.chi2_before,   it.chi2_after, it.lambda,
                 it.pcg_iterations,  it.pcg_converged, it.pcg_relative_residual,
                 it.low_quality_step, it.precond_fallback_blocks, it.accepted, it.wall_seconds};
    }
  }
}

// additive-update vector vertex (toy/circle.hpp:16-28 PointTraits, any dimension)
template <typename FP, int D>
struct VecTraits {
  static constexpr int dimension = D;
  using Vertex = std::array<FP, D>;
  static std::array<FP, D> parameters(const Vertex& v) { return v; }
  static void update(Vertex& v, const FP* delta) {
    for (int k = 0; k < D; ++k) v[k] += delta[k];
  }
  static void set_parameters(Vertex& v, const FP* block) {
    for (int k = 0; k < D; ++k) v[k] = block[k];
  }
};
template <typename FP, int D>
using VecDesc = gopt::VertexDescriptor<FP, FP, VecTraits<FP, D>>;

template <typename FP>
struct CircleTraits {
  static constexpr int residual_dimension = 1;
  using SlotDescriptors = std::tuple<VecDesc<FP, 2>>;
  using Observation = gbm::CircleObs;
  using ConstantData = std::uint8_t;
  template <typename T>
  static void residual(const std::array<const T*, 1>& p, const Observation& o, const ConstantData&, T* e) {
    gbm::circle_residual(p[0], o, e);
  }
};

template <typename FP>
struct StereoTraits {
  static constexpr int residual_dimension = 3;
  using SlotDescriptors = std::tuple<VecDesc<FP, 6>, VecDesc<FP, 3>>;
  using Observation = gbm::StereoObs;
  using ConstantData = gbm::StereoCam;
  template <typename T>
  static void residual(const std::array<const T*, 2>& p, const Observation& o, const ConstantData& k, T* e) {
    gbm::stereo_residual(p[0], p[1], o, k, e);
  }
};

template <typename FP>
struct ImuTraits {
  static constexpr int residual_dimension = 15;
  using SlotDescriptors = std::tuple<VecDesc<FP, 6>, VecDesc<FP, 9>, VecDesc<FP, 6>, VecDesc<FP, 9>>;
  using Observation = gbm::ImuObs;
  using ConstantData = gbm::ImuConst;
  template <typename T>
  static void residual(const std::array<const T*, 4>& p, const Observation& o, const ConstantData& k, T* e) {
    gbm::imu_residual(p[0], p[1], p[2], p[3], o, k, e);
  }
};

template <typename FP, int D>
void load(std::vector<std::array<FP, D>>& dst, const double* src, std::uint64_t n) {
  dst.resize(n);
  for (std::uint64_t i = 0; i < n; ++i)
    for (int k = 0; k < D; ++k) dst[i][k] = static_cast<FP>(src[D * i + k]);
}
template <typename FP, int D>
void store(const std::vector<std::array<FP, D>>& src, double* dst) {
  for (std::size_t i = 0; i < src.size(); ++i)
    for (int k = 0; k < D; ++k) dst[D * i + k] = static_cast<double>(src[i][k]);
}

template <typename FP>
void circle_solve(std::uint64_t n, double* pts, const double* radius, const gb_lm_config& cfg, int workers,
                  gb_solve_report* rep, gb_iteration_record* recs, int max_recs) {
  std::vector<std::array<FP, 2>> v;
  load<FP, 2>(v, pts, n);
  gopt::Graph<FP, FP> graph;
  graph.set_workers(workers);
  VecDesc<FP, 2> vd;
  graph.add_vertex_descriptor(&vd);
  for (std::uint64_t i = 0; i < n; ++i) vd.add_vertex(i, &v[i]);
  gopt::FactorDescriptor<FP, FP, CircleTraits<FP>> fd(&vd);
  fd.set_differentiation_mode(gopt::DifferentiationMode::Auto);
  graph.add_factor_descriptor(&fd);
  for (std::uint64_t i = 0; i < n; ++i) fd.add_factor({i}, gbm::CircleObs{radius[i]}, nullptr, 0, {});
  const gopt::SolveReport r = gopt::levenberg_marquardt(graph, to_lm(cfg));
  store<FP, 2>(v, pts);
  fill(r, rep, recs, max_recs);
}

template <typename FP>
void vi_solve(std::uint64_t npose, double* poses, const std::uint8_t* pose_fixed, std::uint64_t nvb, double* vbs,
              std::uint64_t nlm, double* lms, std::uint64_t nst, const std::uint32_t* st_idx, const double* st_obs,
              const double* cam, std::uint64_t nimu, const std::uint32_t* imu_idx, const double* imu_obs,
              const double* gravity, const gb_lm_config& cfg, int workers, gb_solve_report* rep,
              gb_iteration_record* recs, int max_recs) {
  std::vector<std::array<FP, 6>> P;
  std::vector<std::array<FP, 9>> V;
  std::vector<std::array<FP, 3>> X;
  load<FP, 6>(P, poses, npose);
  load<FP, 9>(V, vbs, nvb);
  load<FP, 3>(X, lms, nlm);
  gopt::Graph<FP, FP> graph;
  graph.set_workers(workers);
  VecDesc<FP, 6> pd;
  VecDesc<FP, 9> vd;
  VecDesc<FP, 3> xd;
  graph.add_vertex_descriptor(&pd);
  graph.add_vertex_descriptor(&vd);
  graph.add_vertex_descriptor(&xd);
  for (std::uint64_t i = 0; i < npose; ++i) {
    pd.add_vertex(i, &P[i]);
    if (pose_fixed && pose_fixed[i]) pd.set_fixed(i, true);
  }
  for (std::uint64_t i = 0; i < nvb; ++i) vd.add_vertex(i, &V[i]);
  for (std::uint64_t i = 0; i < nlm; ++i) xd.add_vertex(i, &X[i]);
  gopt::FactorDescriptor<FP, FP, StereoTraits<FP>> sf(&pd, &xd);
  gopt::FactorDescriptor<FP, FP, ImuTraits<FP>> imf(&pd, &vd, &pd, &vd);
  sf.set_differentiation_mode(gopt::DifferentiationMode::Auto);
  imf.set_differentiation_mode(gopt::DifferentiationMode::Auto);
  graph.add_factor_descriptor(&sf);
  graph.add_factor_descriptor(&imf);
  const gbm::StereoCam k{cam[0], cam[1], cam[2], cam[3], cam[4]};
  for (std::uint64_t i = 0; i < nst; ++i)
    sf.add_factor({st_idx[2 * i], st_idx[2 * i + 1]},
                  gbm::StereoObs{st_obs[3 * i], st_obs[3 * i + 1], st_obs[3 * i + 2]}, nullptr, k, {});
  const gbm::ImuConst g{{gravity[0], gravity[1], gravity[2]}};
  for (std::uint64_t i = 0; i < nimu; ++i) {
    gbm::ImuObs o;
    const double* s = imu_obs + 19 * i;
    for (int q = 0; q < 3; ++q) {
      o.dp[q] = s[q];
      o.dv[q] = s[3 + q];
    }
    for (int q = 0; q < 9; ++q) o.dR[q] = s[6 + q];
    o.dt = s[15];
    imf.add_factor({imu_idx[4 * i], imu_idx[4 * i + 1], imu_idx[4 * i + 2], imu_idx[4 * i + 3]}, o, nullptr, g, {});
  }
  const gopt::SolveReport r = gopt::levenberg_marquardt(graph, to_lm(cfg));
  store<FP, 6>(P, poses);
  store<FP, 9>(V, vbs);
  store<FP, 3>(X, lms);
  fill(r, rep, recs, max_recs);
}

}  // namespace

extern "C" {

const char* refg_last_error(void) { return g_err.c_str(); }

int refg_circle_solve(int precision, uint64_t n, double* points, const double* radius, const gb_lm_config* cfg,
                      int workers, gb_solve_report* rep, gb_iteration_record* recs, int max_recs) {
  return guarded([&] {
    if (precision == GB_FP64)
      circle_solve<double>(n, points, radius, *cfg, workers, rep, recs, max_recs);
    else
      circle_solve<float>(n, points, radius, *cfg, workers, rep, recs, max_recs);
  });
}

int refg_vi_solve(int precision, uint64_t npose, double* poses, const uint8_t* pose_fixed, uint64_t nvb, double* vbs,
                  uint64_t nlm, double* lms, uint64_t nst, const uint32_t* st_idx, const double* st_obs,
                  const double* cam, uint64_t nimu, const uint32_t* imu_idx, const double* imu_obs,
                  const double* gravity, const gb_lm_config* cfg, int workers, gb_solve_report* rep,
                  gb_iteration_record* recs, int max_recs) {
  return guarded([&] {
    if (precision == GB_FP64)
      vi_solve<double>(npose, poses, pose_fixed, nvb, vbs, nlm, lms, nst, st_idx, st_obs, cam, nimu, imu_idx, imu_obs,
                       gravity, *cfg, workers, rep, recs, max_recs);
    else
      vi_solve<float>(npose, poses, pose_fixed, nvb, vbs, nlm, lms, nst, st_idx, st_obs, cam, nimu, imu_idx, imu_obs,
                      gravity, *cfg, workers, rep, recs, max_recs);
  });
}

}  // extern "C"
