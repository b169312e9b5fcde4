// Reference-style client code (the reference README "Library example" and
// src/experiment.cpp:73-80 run_typed, BAL branch) compiled unchanged against
// the B200 facade: -I include/gopt_b200 -I include, linked to libgb_bal.so.
#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <string>

#include "gopt/bal/adapter.hpp"
#include "gopt/levenberg_marquardt.hpp"
#include "gopt/report.hpp"

extern "C" int gb_synthetic_bal(uint64_t, uint64_t, uint64_t, uint64_t, uint64_t, double, uint32_t*, uint32_t*,
                                double*, double*, double*);

template <typename FP, typename SP>
int run(const gopt::bal::BALProblem& problem, const char* name) {
  auto bg = gopt::bal::build_graph<FP, SP>(problem, gopt::DifferentiationMode::Analytic);
  bg->graph.set_workers(8);
  const double mse0 = static_cast<double>(bg->mse());
  gopt::LMConfig lm;
  lm.max_iterations = 50;
  lm.pcg.max_iterations = 10;
  const gopt::SolveReport report = gopt::levenberg_marquardt(bg->graph, lm);
  const double mse1 = static_cast<double>(bg->mse());
  std::printf("%s iterations=%zu accepted=%d termination=%s initial_chi2=%.17g final_chi2=%.17g mse0=%.17g mse1=%.17g "
              "cam0=%.17g pt0=%.17g\n",
              name, report.iterations.size(), report.accepted_steps, gopt::to_string(report.termination),
              report.initial_chi2, report.final_chi2, mse0, mse1, static_cast<double>(bg->cameras[0][0]),
              static_cast<double>(bg->points[0][0]));
  // report wire format (report.hpp:32-71)
  const std::string csv = gopt::to_csv(report);
#ifdef GOPT_B200_HAVE_JSON
  const std::string js = gopt::to_json(report).dump();
  if (js != gopt::to_json_string(report)) return 3;
#else
  const std::string js = gopt::to_json_string(report);
#endif
  std::printf("%s-report csv_lines=%zu json_bytes=%zu\n", name,
              static_cast<size_t>(std::count(csv.begin(), csv.end(), '\n')), js.size());
  return 0;
}

int main() {
  const uint64_t nc = 49, np = 7776, ne = 31843;
  std::vector<uint32_t> ci(ne), pi(ne);
  std::vector<double> obs(2 * ne), cams(9 * nc), pts(3 * np);
  if (gb_synthetic_bal(nc, np, ne, 42, 0, 0.0, ci.data(), pi.data(), obs.data(), cams.data(), pts.data()) != 0)
    return 2;
  gopt::bal::BALProblem p;
  p.cameras.resize(nc);
  p.points.resize(np);
  for (uint64_t c = 0; c < nc; ++c)
    for (int k = 0; k < 9; ++k) p.cameras[c][k] = cams[9 * c + k];
  for (uint64_t q = 0; q < np; ++q)
    for (int k = 0; k < 3; ++k) p.points[q][k] = pts[3 * q + k];
  for (uint64_t i = 0; i < ne; ++i) p.observations.push_back({ci[i], pi[i], obs[2 * i], obs[2 * i + 1]});
  try {
    if (run<double, double>(p, "fp64") || run<float, float>(p, "fp32") || run<float, gopt::bfloat16>(p, "fp32-bf16"))
      return 3;
  } catch (const std::exception& e) {
    std::printf("error: %s\n", e.what());
    return 1;
  }
  return 0;
}
