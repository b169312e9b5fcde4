// ref_capi.cpp — TEST INFRASTRUCTURE ONLY (the parity oracle and the CPU
// baseline). Compiles the UNMODIFIED reference headers from
// /root/reference/proj/include (plus src/bal_problem.cpp) against the
// Eigen-subset shim in oracle/eigen_shim, and exposes the same C ABI as
// include/gb_bal.h with a `ref_` prefix and an extra `workers` argument
// (Graph::set_workers, graph.hpp:50). Nothing here is product code; only
// tests/, __graft_entry__.smoke() and bench.py's CPU legs load the built
// library (oracle/_ref/libgopt_ref.so).
//
// The two private members read here (FactorDescriptor::jblocks_ and
// ::incidence_, factor_descriptor.hpp:772-773) are exposed with the
// `#define private public` trick from a test-only translation unit, as
// SURVEY.md §7 step 0 suggests, so the CSR can be compared bit for bit.

// Every standard header the reference pulls in, first, so the access trick
// below cannot leak into the standard library.
#include <algorithm>
#include <array>
#include <bit>
#include <chrono>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <limits>
#include <memory>
#include <optional>
#include <random>
#include <span>
#include <stdexcept>
#include <string>
#include <thread>
#include <tuple>
#include <type_traits>
#include <unordered_map>
#include <utility>
#include <vector>

#include <Eigen/Dense>

#define private public
#include "gopt/bal/adapter.hpp"
#include "gopt/levenberg_marquardt.hpp"
#undef private

#include "gb_bal.h"

#if __has_include("json.hpp")
#include "gopt/report.hpp"
#define GB_REF_REPORT 1
#endif

namespace {

thread_local std::string g_err;

int set_err(int code, const char* what) {
  g_err = what;
  return code;
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    g_err.clear();
    return GB_OK;
  } catch (const std::invalid_argument& e) {
    return set_err(GB_ERR_INVALID_ARGUMENT, e.what());
  } catch (const std::out_of_range& e) {
    return set_err(GB_ERR_OUT_OF_RANGE, e.what());
  } catch (const std::logic_error& e) {
    return set_err(GB_ERR_LOGIC, e.what());
  } catch (const std::runtime_error& e) {
    return set_err(GB_ERR_RUNTIME, e.what());
  } catch (const std::exception& e) {
    return set_err(GB_ERR_RUNTIME, e.what());
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

gopt::DifferentiationMode to_mode(int m) {
  switch (m) {
    case GB_ANALYTIC: return gopt::DifferentiationMode::Analytic;
    case GB_AUTO: return gopt::DifferentiationMode::Auto;
    case GB_DYNAMIC: return gopt::DifferentiationMode::Dynamic;
  }
  throw std::invalid_argument("unknown differentiation mode");
}

struct RefBase {
  virtual ~RefBase() = default;
  int precision = GB_FP64;
  int diff_mode = GB_ANALYTIC;
  int workers = 1;
  void* user_cams = nullptr;
  void* user_pts = nullptr;
  std::uint64_t nc = 0, np = 0, ne = 0;
  std::vector<std::uint8_t> cam_fixed, pt_fixed, level;
  std::vector<std::uint32_t> cam_idx, pt_idx;
  std::vector<double> obs;  // binary64 BALProblem observations
  int loss_kind = GB_LOSS_DEFAULT;
  double huber = 1.0;
  bool dirty = true;

  virtual void optimize(const gb_lm_config& cfg, gb_solve_report* rep, gb_iteration_record* recs,
                        int max_recs) = 0;
  virtual double mse() = 0;
  virtual double total_error(int level) = 0;
  virtual void ls_linearize(int level, double cmin, double cmax, int damping, double* chi2,
                            std::int64_t* n, void* b, void* diag, void* clamped, void* scaling,
                            std::int32_t* finite) = 0;
  virtual void ls_hvp(const void* v, void* out, double lambda) = 0;
  virtual void ls_precond(double lambda, void* blocks, std::int32_t* fallbacks) = 0;
  virtual void ls_solve_step(double lambda, const gb_pcg_config& pcg, void* dx, gb_pcg_stats* st,
                             double* pred, std::int32_t* finite) = 0;
  virtual void ls_jacobians(void* out) = 0;
  virtual void incidence(int which, std::uint64_t* nseg, std::uint64_t* nitems, std::uint64_t* vos,
                         std::uint64_t* off, std::uint32_t* itf, std::uint16_t* its) = 0;
};

template <typename FP, typename SP>
struct RefImpl final : RefBase {
  std::unique_ptr<gopt::bal::BalGraph<FP, SP>> bg;
  std::unique_ptr<gopt::LinearSystem<FP, SP>> ls;

  void build() {
    if (!dirty && bg) return;
    if (!user_cams || !user_pts) throw std::logic_error("cameras and points must be set first");
    gopt::bal::BALProblem p;
    p.cameras.resize(nc);
    p.points.resize(np);
    const FP* uc = static_cast<const FP*>(user_cams);
    const FP* up = static_cast<const FP*>(user_pts);
    for (std::uint64_t c = 0; c < nc; ++c)
      for (int k = 0; k < 9; ++k) p.cameras[c][k] = static_cast<double>(uc[c * 9 + k]);
    for (std::uint64_t q = 0; q < np; ++q)
      for (int k = 0; k < 3; ++k) p.points[q][k] = static_cast<double>(up[q * 3 + k]);
    p.observations.resize(ne);
    for (std::uint64_t i = 0; i < ne; ++i)
      p.observations[i] = {cam_idx[i], pt_idx[i], obs[2 * i], obs[2 * i + 1]};
    std::optional<double> hub;
    if (loss_kind == GB_LOSS_HUBER) hub = huber;
    bg = gopt::bal::build_graph<FP, SP>(p, to_mode(diff_mode), hub);
    for (std::uint64_t c = 0; c < nc; ++c)
      if (!cam_fixed.empty() && cam_fixed[c]) bg->camera_desc->set_fixed(c, true);
    for (std::uint64_t q = 0; q < np; ++q)
      if (!pt_fixed.empty() && pt_fixed[q]) bg->point_desc->set_fixed(q, true);
    if (!level.empty())
      for (std::uint64_t i = 0; i < ne; ++i)
        if (level[i]) bg->factor_desc->set_level(i, level[i]);
    bg->graph.set_workers(workers);
    ls.reset();
    dirty = false;
  }

  void write_back() {
    FP* uc = static_cast<FP*>(user_cams);
    FP* up = static_cast<FP*>(user_pts);
    for (std::uint64_t c = 0; c < nc; ++c)
      for (int k = 0; k < 9; ++k) uc[c * 9 + k] = bg->cameras[c][k];
    for (std::uint64_t q = 0; q < np; ++q)
      for (int k = 0; k < 3; ++k) up[q * 3 + k] = bg->points[q][k];
  }

  void optimize(const gb_lm_config& cfg, gb_solve_report* rep, gb_iteration_record* recs,
                int max_recs) override {
    dirty = true;  // re-read user parameters
    build();
    const gopt::SolveReport r = gopt::levenberg_marquardt(bg->graph, to_lm(cfg));
    write_back();
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
      rep->memory = {r.memory.jacobian_bytes, r.memory.preconditioner_bytes, r.memory.workspace_bytes,
                     r.memory.graph_bytes};
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

  double mse() override {
    dirty = true;
    build();
    return static_cast<double>(bg->mse());
  }

  double total_error(int lvl) override {
    dirty = true;
    build();
    return static_cast<double>(bg->graph.total_error(lvl));
  }

  void ls_linearize(int lvl, double cmin, double cmax, int damping, double* chi2, std::int64_t* n,
                    void* b, void* diag, void* clamped, void* scaling, std::int32_t* finite) override {
    dirty = true;
    build();
    bg->graph.activate(lvl);
    gopt::LinearSystemOptions opts;
    opts.clamp_min = cmin;
    opts.clamp_max = cmax;
    opts.damping = damping == GB_DAMPING_BEFORE_SCALING ? gopt::DampingPlacement::before_scaling
                                                        : gopt::DampingPlacement::after_scaling;
    ls = std::make_unique<gopt::LinearSystem<FP, SP>>(bg->graph, opts);
    ls->prepare();
    const FP c = ls->linearize();
    if (chi2) *chi2 = static_cast<double>(c);
    if (n) *n = static_cast<std::int64_t>(ls->dims());
    auto cp = [](std::span<const FP> s, void* dst) {
      if (dst) std::memcpy(dst, s.data(), s.size() * sizeof(FP));
    };
    cp(ls->gradient(), b);
    cp(ls->hessian_diagonal(), diag);
    cp(ls->clamped_diagonal(), clamped);
    cp(ls->column_scaling(), scaling);
    if (finite) *finite = ls->linearization_finite() ? 1 : 0;
  }

  void need_ls() const {
    if (!ls) throw std::logic_error("linear system not linearized (call ref_ls_linearize first)");
  }

  void ls_hvp(const void* v, void* out, double lambda) override {
    need_ls();
    using Arith = gopt::arith_t<SP>;
    const std::size_t n = ls->dims();
    ls->hvp(std::span<const SP>(static_cast<const SP*>(v), n), std::span<Arith>(static_cast<Arith*>(out), n),
            static_cast<FP>(lambda));
  }

  void ls_precond(double lambda, void* blocks, std::int32_t* fallbacks) override {
    need_ls();
    ls->build_preconditioner(static_cast<FP>(lambda));
    const auto s = ls->preconditioner_storage();
    if (blocks) std::memcpy(blocks, s.data(), s.size() * sizeof(FP));
    if (fallbacks) *fallbacks = ls->fallback_blocks();
  }

  void ls_solve_step(double lambda, const gb_pcg_config& pcg, void* dx, gb_pcg_stats* st, double* pred,
                     std::int32_t* finite) override {
    need_ls();
    gopt::PCGConfig c;
    c.max_iterations = pcg.max_iterations;
    c.tolerance = pcg.tolerance;
    c.rejection_ratio = pcg.rejection_ratio;
    c.normalize_rhs = pcg.normalize_rhs != 0;
    std::vector<FP> out(ls->dims());
    const auto r = ls->solve_step(static_cast<FP>(lambda), c, out);
    if (dx) std::memcpy(dx, out.data(), out.size() * sizeof(FP));
    if (st) *st = {r.stats.iterations, r.stats.final_relative_residual, r.stats.converged ? 1 : 0};
    if (pred) *pred = static_cast<double>(r.predicted_decrease);
    if (finite) *finite = r.finite ? 1 : 0;
  }

  void ls_jacobians(void* out) override {
    need_ls();
    const auto& jb = bg->factor_desc->jblocks_;
    if (out) std::memcpy(out, jb.data(), jb.size() * sizeof(SP));
  }

  void incidence(int which, std::uint64_t* nseg, std::uint64_t* nitems, std::uint64_t* vos,
                 std::uint64_t* off, std::uint32_t* itf, std::uint16_t* its) override {
    need_ls();
    const auto& incs = bg->factor_desc->incidence_;
    if (which < 0 || which >= static_cast<int>(incs.size())) throw std::out_of_range("incidence index");
    const auto& inc = incs[static_cast<std::size_t>(which)];
    if (nseg) *nseg = inc.vertex_of_segment.size();
    if (nitems) *nitems = inc.items.size();
    if (vos)
      for (std::size_t i = 0; i < inc.vertex_of_segment.size(); ++i) vos[i] = inc.vertex_of_segment[i];
    if (off)
      for (std::size_t i = 0; i < inc.offsets.size(); ++i) off[i] = inc.offsets[i];
    if (itf || its)
      for (std::size_t i = 0; i < inc.items.size(); ++i) {
        if (itf) itf[i] = inc.items[i].first;
        if (its) its[i] = inc.items[i].second;
      }
  }
};

}  // namespace

extern "C" {

struct ref_graph {
  std::unique_ptr<RefBase> impl;
};

const char* ref_last_error(void) { return g_err.c_str(); }

ref_graph* ref_create(int precision, int diff_mode, int workers) {
  auto* g = new ref_graph;
  switch (precision) {
    case GB_FP64: g->impl = std::make_unique<RefImpl<double, double>>(); break;
    case GB_FP32: g->impl = std::make_unique<RefImpl<float, float>>(); break;
    case GB_FP32_BF16: g->impl = std::make_unique<RefImpl<float, gopt::bfloat16>>(); break;
    default:
      delete g;
      set_err(GB_ERR_INVALID_ARGUMENT, "invalid precision");
      return nullptr;
  }
  g->impl->precision = precision;
  g->impl->diff_mode = diff_mode;
  g->impl->workers = workers < 1 ? 1 : workers;
  return g;
}

void ref_destroy(ref_graph* g) { delete g; }

int ref_set_workers(ref_graph* g, int workers) {
  g->impl->workers = workers < 1 ? 1 : workers;
  g->impl->dirty = true;
  return GB_OK;
}

int ref_set_cameras(ref_graph* g, void* params, std::uint64_t n, const std::uint8_t* fixed) {
  g->impl->user_cams = params;
  g->impl->nc = n;
  g->impl->cam_fixed.assign(fixed ? fixed : nullptr, fixed ? fixed + n : nullptr);
  g->impl->dirty = true;
  return GB_OK;
}

int ref_set_points(ref_graph* g, void* params, std::uint64_t n, const std::uint8_t* fixed) {
  g->impl->user_pts = params;
  g->impl->np = n;
  g->impl->pt_fixed.assign(fixed ? fixed : nullptr, fixed ? fixed + n : nullptr);
  g->impl->dirty = true;
  return GB_OK;
}

int ref_set_observations(ref_graph* g, std::uint64_t n, const std::uint32_t* cam, const std::uint32_t* pt,
                         const void* observed, const std::uint8_t* level, int loss_kind,
                         double huber_delta) {
  RefBase& b = *g->impl;
  b.ne = n;
  b.cam_idx.assign(cam, cam + n);
  b.pt_idx.assign(pt, pt + n);
  b.obs.resize(2 * n);
  if (b.precision == GB_FP64) {
    const double* o = static_cast<const double*>(observed);
    std::copy(o, o + 2 * n, b.obs.begin());
  } else {
    const float* o = static_cast<const float*>(observed);
    for (std::uint64_t i = 0; i < 2 * n; ++i) b.obs[i] = o[i];
  }
  b.level.assign(level ? level : nullptr, level ? level + n : nullptr);
  b.loss_kind = loss_kind;
  b.huber = huber_delta;
  b.dirty = true;
  return GB_OK;
}

int ref_optimize(ref_graph* g, const gb_lm_config* cfg, gb_solve_report* rep, gb_iteration_record* recs,
                 std::int32_t max_recs) {
  return guarded([&] { g->impl->optimize(*cfg, rep, recs, max_recs); });
}

int ref_mse(ref_graph* g, double* out) {
  return guarded([&] { *out = g->impl->mse(); });
}

int ref_total_error(ref_graph* g, int level, double* out) {
  return guarded([&] { *out = g->impl->total_error(level); });
}

int ref_ls_linearize(ref_graph* g, int level, double cmin, double cmax, int damping, double* chi2,
                     std::int64_t* n, void* b, void* diag, void* clamped, void* scaling,
                     std::int32_t* finite) {
  return guarded([&] { g->impl->ls_linearize(level, cmin, cmax, damping, chi2, n, b, diag, clamped, scaling, finite); });
}

int ref_ls_hvp(ref_graph* g, const void* v, void* out, double lambda) {
  return guarded([&] { g->impl->ls_hvp(v, out, lambda); });
}

int ref_ls_preconditioner(ref_graph* g, double lambda, void* blocks, std::int32_t* fallbacks) {
  return guarded([&] { g->impl->ls_precond(lambda, blocks, fallbacks); });
}

int ref_ls_solve_step(ref_graph* g, double lambda, const gb_pcg_config* pcg, void* dx, gb_pcg_stats* st,
                      double* pred, std::int32_t* finite) {
  return guarded([&] { g->impl->ls_solve_step(lambda, *pcg, dx, st, pred, finite); });
}

int ref_ls_jacobians(ref_graph* g, void* out) {
  return guarded([&] { g->impl->ls_jacobians(out); });
}

int ref_incidence(ref_graph* g, int which, std::uint64_t* nseg, std::uint64_t* nitems, std::uint64_t* vos,
                  std::uint64_t* off, std::uint32_t* itf, std::uint16_t* its) {
  return guarded([&] { g->impl->incidence(which, nseg, nitems, vos, off, itf, its); });
}

// Snavely closed forms (bal/snavely.hpp:18-153) at binary64, for the
// known-answer and finite-difference suites (tests/test_bal.cpp:120-276).
void ref_snavely_project(const double* camera, const double* point, double* predicted) {
  gopt::bal::snavely_project<double>(camera, point, predicted);
}
void ref_rotate_angle_axis(const double* omega, const double* x, double* y) {
  gopt::bal::rotate_angle_axis<double>(omega, x, y);
}
void ref_snavely_jacobians(const double* camera, const double* point, double* jc, double* jp) {
  gopt::bal::snavely_camera_jacobian<double>(camera, point, jc);
  gopt::bal::snavely_point_jacobian<double>(camera, point, jp);
}
// Nielsen schedule (levenberg_marquardt.hpp:88-98).
void ref_update_damping(double* lambda, double* nu, int accepted, double gain) {
  gopt::update_damping<double>(*lambda, *nu, accepted != 0, gain);
}
// bfloat16 RNE narrowing (bfloat16.hpp:25-33).
std::uint16_t ref_bf16_round(float f) { return gopt::bfloat16::round_from(f); }

// bal::parse_bal_file (src/bal_problem.cpp:81-119): reads a BAL text file with
// the reference's own tokenizer. Call once with NULL outputs to get the shape,
// then again with arrays of that size.
int ref_parse_bal_file(const char* path, std::uint64_t* shape3, std::uint32_t* cam, std::uint32_t* pt,
                       double* obs, double* cams, double* pts) {
  return guarded([&] {
    const gopt::bal::BALProblem p = gopt::bal::parse_bal_file(path);
    shape3[0] = p.num_cameras();
    shape3[1] = p.num_points();
    shape3[2] = p.num_observations();
    if (!cam) return;
    for (std::size_t i = 0; i < p.observations.size(); ++i) {
      cam[i] = p.observations[i].camera_index;
      pt[i] = p.observations[i].point_index;
      obs[2 * i] = p.observations[i].x;
      obs[2 * i + 1] = p.observations[i].y;
    }
    for (std::size_t c = 0; c < p.cameras.size(); ++c)
      for (int k = 0; k < 9; ++k) cams[9 * c + k] = p.cameras[c][k];
    for (std::size_t q = 0; q < p.points.size(); ++q)
      for (int k = 0; k < 3; ++k) pts[3 * q + k] = p.points[q][k];
  });
}

#ifdef GB_REF_REPORT
// gopt::to_json(report).dump() / gopt::to_csv(report) (report.hpp:32-71) of a
// SolveReport rebuilt from the C structs
static gopt::SolveReport from_c(const gb_solve_report* r, const gb_iteration_record* recs, int n) {
  gopt::SolveReport s;
  for (int i = 0; i < n; ++i) {
    gopt::IterationRecord x;
    x.iteration = recs[i].iteration;
    x.chi2_before = recs[i].chi2_before;
    x.chi2_after = recs[i].chi2_after;
    x.lambda = recs[i].lambda;
    x.pcg_iterations = recs[i].pcg_iterations;
    x.pcg_converged = recs[i].pcg_converged != 0;
    x.pcg_relative_residual = recs[i].pcg_relative_residual;
    x.low_quality_step = recs[i].low_quality_step != 0;
    x.precond_fallback_blocks = recs[i].precond_fallback_blocks;
    x.accepted = recs[i].accepted != 0;
    x.wall_seconds = recs[i].wall_seconds;
    s.iterations.push_back(x);
  }
  s.initial_chi2 = r->initial_chi2;
  s.final_chi2 = r->final_chi2;
  s.accepted_steps = r->accepted_steps;
  s.termination = static_cast<gopt::Termination>(r->termination);
  s.total_seconds = r->total_seconds;
  s.free_dims = r->free_dims;
  s.residual_dims = r->residual_dims;
  s.active_factors = r->active_factors;
  s.memory.jacobian_bytes = r->memory.jacobian_bytes;
  s.memory.preconditioner_bytes = r->memory.preconditioner_bytes;
  s.memory.workspace_bytes = r->memory.workspace_bytes;
  s.memory.graph_bytes = r->memory.graph_bytes;
  return s;
}
static int emit(const std::string& s, char* buf, std::uint64_t cap, std::uint64_t* needed) {
  if (needed) *needed = s.size() + 1;
  if (buf && cap) {
    const std::size_t n = std::min<std::uint64_t>(cap - 1, s.size());
    std::memcpy(buf, s.data(), n);
    buf[n] = '\0';
  }
  return GB_OK;
}
int ref_report_json(const gb_solve_report* r, const gb_iteration_record* recs, std::int32_t n, char* buf,
                    std::uint64_t cap, std::uint64_t* needed) {
  return emit(gopt::to_json(from_c(r, recs, n)).dump(), buf, cap, needed);
}
int ref_report_csv(const gb_solve_report* r, const gb_iteration_record* recs, std::int32_t n, char* buf,
                   std::uint64_t cap, std::uint64_t* needed) {
  return emit(gopt::to_csv(from_c(r, recs, n)), buf, cap, needed);
}
#endif

}  // extern "C"
