// Drop-in for the reference header gopt/report.hpp (include/gopt/report.hpp:11-73):
// to_json / to_csv of a SolveReport. The bytes come from the product's C ABI
// (gb_report_json / gb_report_csv, identical to the reference's output);
// to_json returns an nlohmann::json when the client has nlohmann/json on its
// include path (the reference includes it as "json.hpp"), so
// to_json(report).dump() reproduces the reference's string.
#pragma once

#include <string>
#include <vector>

#include "../gopt.hpp"

namespace gopt {
namespace detail {
inline void report_to_c(const SolveReport& r, gb_solve_report* c, std::vector<gb_iteration_record>* recs) {
  *c = gb_solve_report{};
  c->initial_chi2 = r.initial_chi2;
  c->final_chi2 = r.final_chi2;
  c->accepted_steps = r.accepted_steps;
  c->termination = static_cast<int32_t>(r.termination);
  c->total_seconds = r.total_seconds;
  c->free_dims = r.free_dims;
  c->residual_dims = r.residual_dims;
  c->active_factors = r.active_factors;
  c->memory = {r.memory.jacobian_bytes, r.memory.preconditioner_bytes, r.memory.workspace_bytes, r.memory.graph_bytes};
  c->iterations_run = static_cast<int32_t>(r.iterations.size());
  recs->clear();
  for (const IterationRecord& x : r.iterations)
    recs->push_back({x.iteration, x.chi2_before, x.chi2_after, x.lambda, x.pcg_iterations, x.pcg_converged ? 1 : 0,
                     x.pcg_relative_residual, x.low_quality_step ? 1 : 0, x.precond_fallback_blocks,
                     x.accepted ? 1 : 0, x.wall_seconds});
}
template <typename F>
std::string report_bytes(const SolveReport& r, F fn) {
  gb_solve_report c;
  std::vector<gb_iteration_record> recs;
  report_to_c(r, &c, &recs);
  uint64_t need = 0;
  check(fn(&c, recs.data(), static_cast<int32_t>(recs.size()), nullptr, 0, &need));
  std::string s(need, '\0');
  check(fn(&c, recs.data(), static_cast<int32_t>(recs.size()), s.data(), need, nullptr));
  s.resize(need - 1);
  return s;
}
}  // namespace detail

/// report.hpp:51-71 (fixed CSV column order, '#' summary header lines)
inline std::string to_csv(const SolveReport& report) { return detail::report_bytes(report, gb_report_csv); }

/// to_json(report).dump() of report.hpp:32-47 as a string
inline std::string to_json_string(const SolveReport& report) {
  return detail::report_bytes(report, gb_report_json);
}

}  // namespace gopt

#if __has_include("json.hpp")
#include "json.hpp"
#define GOPT_B200_HAVE_JSON 1
#elif __has_include(<nlohmann/json.hpp>)
#include <nlohmann/json.hpp>
#define GOPT_B200_HAVE_JSON 1
#endif

#ifdef GOPT_B200_HAVE_JSON
namespace gopt {
/// report.hpp:32-47
inline nlohmann::json to_json(const SolveReport& report) { return nlohmann::json::parse(to_json_string(report)); }
}  // namespace gopt
#endif
