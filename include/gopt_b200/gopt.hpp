// gopt_b200/gopt.hpp — drop-in C++ facade for the reference's LM path.
//
// Code written against the reference (`#include "gopt/bal/adapter.hpp"`,
// `gopt::levenberg_marquardt(graph, config)`, /root/reference/proj/README.md
// "Library example") compiles unchanged against this header and runs the
// solve on the B200 through the C ABI (include/gb_bal.h). Same namespace,
// type names, field names, defaults and exception types as the reference:
//
//   gopt::ScalarKind / PrecisionPair / bfloat16     precision.hpp, bfloat16.hpp
//   gopt::LossKind / LossParams<FP>                  loss.hpp:10-23
//   gopt::DifferentiationMode / DampingPlacement     factor_descriptor.hpp:23-37
//   gopt::PCGConfig / PCGStats                       pcg.hpp:12-23
//   gopt::LinearSystemOptions                        linear_system.hpp:15-19
//   gopt::LMConfig / Termination / IterationRecord /
//         MemoryAccount / SolveReport / update_damping levenberg_marquardt.hpp:15-98
//   gopt::VertexDescriptor<FP,SP,Traits>             vertex_descriptor.hpp:57-177
//   gopt::FactorDescriptor<FP,SP,Traits>             factor_descriptor.hpp:152-774
//   gopt::Graph<FP,SP>                               graph.hpp:26-164
//   gopt::levenberg_marquardt<FP,SP>                 levenberg_marquardt.hpp:115-224
//   gopt::bal::{CameraTraits, Point3Traits, ReprojectionTraits, CameraDescriptor,
//     Point3Descriptor, ReprojectionFactor, BalGraph, build_graph, BALProblem}
//                                                    bal/adapter.hpp, bal/problem.hpp
//
// Scope (tier framing): the device path is the BAL graph — one
// camera descriptor, one point descriptor, one reprojection factor
// descriptor, identity information, one loss for all factors. Any other graph
// throws std::invalid_argument; there is no CPU fallback.
#pragma once

#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <tuple>
#include <type_traits>
#include <unordered_map>
#include <vector>

#include "gb_bal.h"

namespace gopt {

// ------------------------------------------------------------- precision
enum class ScalarKind { binary64, binary32, bfloat16_storage };

struct bfloat16 {
  std::uint16_t bits = 0;
  bfloat16() = default;
  explicit bfloat16(float f) {
    std::uint32_t u;
    std::memcpy(&u, &f, 4);
    if (std::isnan(f)) {
      bits = static_cast<std::uint16_t>(((u >> 16) & 0x8000u) | 0x7FC0u);
    } else {
      bits = static_cast<std::uint16_t>((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
    }
  }
  explicit operator float() const {
    const std::uint32_t u = static_cast<std::uint32_t>(bits) << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
  }
};

template <typename T>
struct scalar_kind_of;
template <>
struct scalar_kind_of<double> {
  static constexpr ScalarKind value = ScalarKind::binary64;
};
template <>
struct scalar_kind_of<float> {
  static constexpr ScalarKind value = ScalarKind::binary32;
};
template <>
struct scalar_kind_of<bfloat16> {
  static constexpr ScalarKind value = ScalarKind::bfloat16_storage;
};

struct PrecisionPair {
  ScalarKind graph_precision = ScalarKind::binary64;
  ScalarKind system_precision = ScalarKind::binary64;
};

namespace detail {
template <typename FP, typename SP>
constexpr int precision_code() {
  if constexpr (std::is_same_v<FP, double> && std::is_same_v<SP, double>) return GB_FP64;
  else if constexpr (std::is_same_v<FP, float> && std::is_same_v<SP, float>) return GB_FP32;
  else if constexpr (std::is_same_v<FP, float> && std::is_same_v<SP, bfloat16>) return GB_FP32_BF16;
  else return -1;
}

inline void check(int rc) {
  if (rc == GB_OK) return;
  const std::string msg = gb_last_error();
  switch (rc) {
    case GB_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case GB_ERR_OUT_OF_RANGE: throw std::out_of_range(msg);
    case GB_ERR_LOGIC: throw std::logic_error(msg);
    default: throw std::runtime_error(msg);
  }
}
}  // namespace detail

// -------------------------------------------------------------- loss
enum class LossKind { Default, Huber };

template <typename FP>
struct LossParams {
  LossKind kind = LossKind::Default;
  FP delta = FP(1);
  static LossParams Default() { return {LossKind::Default, FP(1)}; }
  static LossParams Huber(FP delta) { return {LossKind::Huber, delta}; }
};

enum class DifferentiationMode { Analytic, Auto, Dynamic };
enum class DampingPlacement { after_scaling, before_scaling };

// ------------------------------------------------------------ configs
struct PCGConfig {
  int max_iterations = 50;
  double tolerance = 1e-6;
  double rejection_ratio = 10.0;
  bool normalize_rhs = true;
};

struct PCGStats {
  int iterations = 0;
  double final_relative_residual = 0.0;
  bool converged = false;
};

struct LinearSystemOptions {
  double clamp_min = 1e-6;
  double clamp_max = 1e32;
  DampingPlacement damping = DampingPlacement::after_scaling;
};

struct LMConfig {
  int max_iterations = 10;
  double tolerance = 1e-6;
  int level = 0;
  double tau = 1e-4;
  PCGConfig pcg;
  LinearSystemOptions linear;
  bool use_rejection_guard = true;
  bool refresh_on_reject = false;
  double lambda_max = 1e32;
  double gradient_tolerance = 1e-12;
};

enum class Termination {
  max_iterations,
  tolerance_reached,
  gradient_small,
  damping_overflow,
  non_finite_linearization,
  no_free_parameters,
};

inline const char* to_string(Termination t) {
  switch (t) {
    case Termination::max_iterations: return "max_iterations";
    case Termination::tolerance_reached: return "tolerance_reached";
    case Termination::gradient_small: return "gradient_small";
    case Termination::damping_overflow: return "damping_overflow";
    case Termination::non_finite_linearization: return "non_finite_linearization";
    case Termination::no_free_parameters: return "no_free_parameters";
  }
  return "?";
}

struct IterationRecord {
  int iteration = 0;
  double chi2_before = 0;
  double chi2_after = 0;
  double lambda = 0;
  int pcg_iterations = 0;
  bool pcg_converged = false;
  double pcg_relative_residual = 0;
  bool low_quality_step = false;
  int precond_fallback_blocks = 0;
  bool accepted = false;
  double wall_seconds = 0;
};

struct MemoryAccount {
  std::size_t jacobian_bytes = 0;
  std::size_t preconditioner_bytes = 0;
  std::size_t workspace_bytes = 0;
  std::size_t graph_bytes = 0;
};

struct SolveReport {
  std::vector<IterationRecord> iterations;
  double initial_chi2 = 0;
  double final_chi2 = 0;
  int accepted_steps = 0;
  Termination termination = Termination::max_iterations;
  double total_seconds = 0;
  std::int64_t free_dims = 0;
  std::int64_t residual_dims = 0;
  std::size_t active_factors = 0;
  MemoryAccount memory;
};

// Nielsen schedule (levenberg_marquardt.hpp:88-98): host-side helper, the
// solve itself runs it on the device.
template <typename FP>
void update_damping(FP& lambda, FP& nu, bool accepted, FP gain_ratio) {
  if (accepted) {
    const FP g = FP(2) * gain_ratio - FP(1);
    lambda *= std::max(FP(1) / FP(3), FP(1) - g * g * g);
    nu = FP(2);
  } else {
    lambda *= nu;
    nu *= FP(2);
  }
}

// -------------------------------------------------------- descriptors
inline constexpr std::int64_t kFixedColumn = -1;

template <typename FP, typename SP>
class VertexDescriptorBase {
 public:
  virtual ~VertexDescriptorBase() = default;
  virtual std::size_t size() const = 0;
  virtual int block_dimension() const = 0;
  virtual bool fixed_at(std::size_t index) const = 0;
  // device bridge: gather parameters AoS into dst, scatter back from src
  virtual void gather(FP* dst) const = 0;
  virtual void scatter(const FP* src) = 0;
};

template <typename FP, typename SP, typename Traits>
class VertexDescriptor final : public VertexDescriptorBase<FP, SP> {
 public:
  using Vertex = typename Traits::Vertex;
  using TraitsType = Traits;
  static constexpr int kDim = Traits::dimension;

  void reserve(std::size_t n) {
    entries_.reserve(n);
    index_.reserve(n);
  }
  void add_vertex(std::uint64_t vertex_id, Vertex* handle) {
    if (handle == nullptr) throw std::invalid_argument("add_vertex: null handle");
    auto [it, inserted] = index_.emplace(vertex_id, entries_.size());
    if (!inserted) throw std::invalid_argument("add_vertex: duplicate vertex id " + std::to_string(vertex_id));
    entries_.push_back({handle, false});
  }
  void set_fixed(std::uint64_t vertex_id, bool fixed) { entries_[position_of(vertex_id)].fixed = fixed; }
  bool is_fixed(std::uint64_t vertex_id) const { return entries_[position_of(vertex_id)].fixed; }
  std::size_t position_of(std::uint64_t vertex_id) const {
    auto it = index_.find(vertex_id);
    if (it == index_.end()) throw std::invalid_argument("unknown vertex id " + std::to_string(vertex_id));
    return it->second;
  }
  std::optional<std::size_t> try_position(std::uint64_t vertex_id) const {
    auto it = index_.find(vertex_id);
    if (it == index_.end()) return std::nullopt;
    return it->second;
  }
  const Vertex& vertex_at(std::size_t i) const { return *entries_[i].handle; }
  std::size_t size() const override { return entries_.size(); }
  int block_dimension() const override { return kDim; }
  bool fixed_at(std::size_t i) const override { return entries_[i].fixed; }
  void gather(FP* dst) const override {
    for (std::size_t i = 0; i < entries_.size(); ++i) {
      const auto block = Traits::parameters(*entries_[i].handle);
      for (int k = 0; k < kDim; ++k) dst[i * kDim + k] = block[k];
    }
  }
  void scatter(const FP* src) override {
    for (std::size_t i = 0; i < entries_.size(); ++i)
      if (!entries_[i].fixed) Traits::set_parameters(*entries_[i].handle, src + i * kDim);
  }

 private:
  struct Entry {
    Vertex* handle;
    bool fixed;
  };
  std::vector<Entry> entries_;
  std::unordered_map<std::uint64_t, std::size_t> index_;
};

template <typename FP, typename SP>
class FactorDescriptorBase {
 public:
  virtual ~FactorDescriptorBase() = default;
  virtual std::size_t size() const = 0;
  virtual DifferentiationMode differentiation_mode() const = 0;
  virtual std::vector<const void*> slot_descriptor_ids() const = 0;
  // device bridge (BAL reprojection factors only)
  virtual bool is_bal_reprojection() const = 0;
  virtual void export_bal(std::vector<std::uint32_t>& cam, std::vector<std::uint32_t>& pt, std::vector<FP>& obs,
                          std::vector<std::uint8_t>& level, int& loss_kind, double& delta) const = 0;
};

template <typename FP, typename SP, typename Traits>
class FactorDescriptor final : public FactorDescriptorBase<FP, SP> {
 public:
  using SlotDescs = typename Traits::SlotDescriptors;
  using Observation = typename Traits::Observation;
  using ConstantData = typename Traits::ConstantData;
  static constexpr std::size_t kArity = std::tuple_size_v<SlotDescs>;
  static constexpr int kResDim = Traits::residual_dimension;
  using SlotPtrs = decltype(std::apply([](auto... d) { return std::tuple<decltype(&d)...>{}; }, SlotDescs{}));

  template <typename... Ds>
  explicit FactorDescriptor(Ds*... slots) : slots_(slots...) {}

  void reserve(std::size_t n) { entries_.reserve(n); }
  void add_factor(const std::array<std::uint64_t, kArity>& ids, Observation observation, const FP* information,
                  ConstantData, LossParams<FP> loss) {
    Entry e;
    resolve(ids, e.slot_pos, std::make_index_sequence<kArity>{});
    e.obs = observation;
    e.loss = loss;
    e.identity = true;
    if (information) {
      for (int i = 0; i < kResDim; ++i)
        for (int j = 0; j < kResDim; ++j)
          if (information[i * kResDim + j] != (i == j ? FP(1) : FP(0))) e.identity = false;
    }
    e.level = 0;
    entries_.push_back(e);
  }
  void set_level(std::size_t index, std::uint8_t level) {
    if (index >= entries_.size())
      throw std::out_of_range("factor index " + std::to_string(index) + " out of range (size " +
                              std::to_string(entries_.size()) + ")");
    entries_[index].level = level;
  }
  void set_differentiation_mode(DifferentiationMode m) { mode_ = m; }
  DifferentiationMode differentiation_mode() const override { return mode_; }
  std::size_t size() const override { return entries_.size(); }
  std::vector<const void*> slot_descriptor_ids() const override {
    std::vector<const void*> out;
    std::apply([&](auto*... d) { (out.push_back(static_cast<const void*>(d)), ...); }, slots_);
    return out;
  }
  bool is_bal_reprojection() const override { return Traits::kIsBalReprojection; }
  void export_bal(std::vector<std::uint32_t>& cam, std::vector<std::uint32_t>& pt, std::vector<FP>& obs,
                  std::vector<std::uint8_t>& level, int& loss_kind, double& delta) const override {
    const std::size_t n = entries_.size();
    cam.resize(n);
    pt.resize(n);
    obs.resize(2 * n);
    level.resize(n);
    loss_kind = GB_LOSS_DEFAULT;
    delta = 1.0;
    for (std::size_t i = 0; i < n; ++i) {
      const Entry& e = entries_[i];
      if (!e.identity) throw std::invalid_argument("device path: non-identity information is not supported");
      const int lk = e.loss.kind == LossKind::Huber ? GB_LOSS_HUBER : GB_LOSS_DEFAULT;
      if (i == 0) {
        loss_kind = lk;
        delta = static_cast<double>(e.loss.delta);
      } else if (lk != loss_kind || (lk == GB_LOSS_HUBER && static_cast<double>(e.loss.delta) != delta)) {
        throw std::invalid_argument("device path: one loss for all factors");
      }
      cam[i] = e.slot_pos[0];
      pt[i] = e.slot_pos[1];
      obs[2 * i] = e.obs[0];
      obs[2 * i + 1] = e.obs[1];
      level[i] = e.level;
    }
  }

 private:
  struct Entry {
    std::array<std::uint32_t, kArity> slot_pos;
    Observation obs;
    LossParams<FP> loss;
    bool identity;
    std::uint8_t level;
  };
  template <std::size_t... Is>
  void resolve(const std::array<std::uint64_t, kArity>& ids, std::array<std::uint32_t, kArity>& out,
               std::index_sequence<Is...>) const {
    (resolve_one<Is>(ids[Is], out[Is]), ...);
  }
  template <std::size_t S>
  void resolve_one(std::uint64_t id, std::uint32_t& out) const {
    auto pos = std::get<S>(slots_)->try_position(id);
    if (!pos)
      throw std::invalid_argument("add_factor: slot " + std::to_string(S) + " references unknown vertex id " +
                                  std::to_string(id));
    out = static_cast<std::uint32_t>(*pos);
  }
  SlotPtrs slots_;
  std::vector<Entry> entries_;
  DifferentiationMode mode_ = DifferentiationMode::Auto;
};

// ------------------------------------------------------------------ graph
template <typename FP, typename SP>
class Graph {
 public:
  static_assert(sizeof(SP) <= sizeof(FP), "system precision must not exceed graph precision");
  static constexpr PrecisionPair precision() { return PrecisionPair{scalar_kind_of<FP>::value, scalar_kind_of<SP>::value}; }

  void add_vertex_descriptor(VertexDescriptorBase<FP, SP>* vd) {
    if (vd == nullptr) throw std::invalid_argument("null vertex descriptor");
    vertex_descs_.push_back(vd);
  }
  void add_factor_descriptor(FactorDescriptorBase<FP, SP>* fd) {
    if (fd == nullptr) throw std::invalid_argument("null factor descriptor");
    factor_descs_.push_back(fd);
  }
  const std::vector<VertexDescriptorBase<FP, SP>*>& vertex_descriptors() const { return vertex_descs_; }
  const std::vector<FactorDescriptorBase<FP, SP>*>& factor_descriptors() const { return factor_descs_; }
  // Graph::set_workers (graph.hpp:50): the device path ignores the CPU worker count.
  void set_workers(int workers) { workers_ = workers < 1 ? 1 : workers; }
  int workers() const { return workers_; }
  void set_device(int device) { device_ = device; }
  int device() const { return device_; }

 private:
  std::vector<VertexDescriptorBase<FP, SP>*> vertex_descs_;
  std::vector<FactorDescriptorBase<FP, SP>*> factor_descs_;
  int workers_ = 1;
  int device_ = 0;
};

namespace detail {
struct Handle {
  gb_graph* g = nullptr;
  ~Handle() {
    if (g) gb_destroy(g);
  }
};

inline int mode_code(DifferentiationMode m) {
  return m == DifferentiationMode::Analytic ? GB_ANALYTIC : m == DifferentiationMode::Auto ? GB_AUTO : GB_DYNAMIC;
}

inline gb_lm_config to_c(const LMConfig& c) {
  gb_lm_config o;
  gb_default_config(&o);
  o.max_iterations = c.max_iterations;
  o.tolerance = c.tolerance;
  o.level = c.level;
  o.tau = c.tau;
  o.pcg.max_iterations = c.pcg.max_iterations;
  o.pcg.tolerance = c.pcg.tolerance;
  o.pcg.rejection_ratio = c.pcg.rejection_ratio;
  o.pcg.normalize_rhs = c.pcg.normalize_rhs ? 1 : 0;
  o.clamp_min = c.linear.clamp_min;
  o.clamp_max = c.linear.clamp_max;
  o.damping = c.linear.damping == DampingPlacement::before_scaling ? GB_DAMPING_BEFORE_SCALING : GB_DAMPING_AFTER_SCALING;
  o.use_rejection_guard = c.use_rejection_guard ? 1 : 0;
  o.refresh_on_reject = c.refresh_on_reject ? 1 : 0;
  o.lambda_max = c.lambda_max;
  o.gradient_tolerance = c.gradient_tolerance;
  return o;
}
}  // namespace detail

// levenberg_marquardt (levenberg_marquardt.hpp:115-224) on the B200.
template <typename FP, typename SP>
SolveReport levenberg_marquardt(Graph<FP, SP>& graph, const LMConfig& config) {
  constexpr int prec = detail::precision_code<FP, SP>();
  static_assert(prec >= 0, "precision pair must be <double,double>, <float,float> or <float,bfloat16>");
  const auto& vds = graph.vertex_descriptors();
  const auto& fds = graph.factor_descriptors();
  if (vds.size() != 2 || fds.size() != 1 || !fds[0]->is_bal_reprojection() || vds[0]->block_dimension() != 9 ||
      vds[1]->block_dimension() != 3)
    throw std::invalid_argument(
        "device path: expects the bal::build_graph structure (cameras, points, one reprojection factor descriptor)");
  const auto ids = fds[0]->slot_descriptor_ids();
  if (ids.size() != 2 || ids[0] != static_cast<const void*>(vds[0]) || ids[1] != static_cast<const void*>(vds[1]))
    throw std::logic_error("factor descriptor references a vertex descriptor not in this graph");

  auto* cams = vds[0];
  auto* pts = vds[1];
  std::vector<FP> cbuf(cams->size() * 9), pbuf(pts->size() * 3);
  cams->gather(cbuf.data());
  pts->gather(pbuf.data());
  std::vector<std::uint8_t> cfix(cams->size()), pfix(pts->size());
  for (std::size_t i = 0; i < cams->size(); ++i) cfix[i] = cams->fixed_at(i) ? 1 : 0;
  for (std::size_t i = 0; i < pts->size(); ++i) pfix[i] = pts->fixed_at(i) ? 1 : 0;
  std::vector<std::uint32_t> ci, pi;
  std::vector<FP> obs;
  std::vector<std::uint8_t> lvl;
  int loss_kind;
  double delta;
  fds[0]->export_bal(ci, pi, obs, lvl, loss_kind, delta);

  detail::Handle h;
  h.g = gb_create(prec, detail::mode_code(fds[0]->differentiation_mode()), graph.device());
  if (!h.g) detail::check(GB_ERR_NO_DEVICE);
  detail::check(gb_set_cameras(h.g, cbuf.data(), cams->size(), cfix.data()));
  detail::check(gb_set_points(h.g, pbuf.data(), pts->size(), pfix.data()));
  detail::check(gb_set_observations(h.g, ci.size(), ci.data(), pi.data(), obs.data(), lvl.data(), loss_kind, delta));
  const gb_lm_config cfg = detail::to_c(config);
  gb_solve_report rep{};
  std::vector<gb_iteration_record> recs(static_cast<std::size_t>(std::max(1, config.max_iterations)));
  detail::check(gb_optimize(h.g, &cfg, &rep, recs.data(), static_cast<std::int32_t>(recs.size())));
  cams->scatter(cbuf.data());
  pts->scatter(pbuf.data());

  SolveReport out;
  out.initial_chi2 = rep.initial_chi2;
  out.final_chi2 = rep.final_chi2;
  out.accepted_steps = rep.accepted_steps;
  out.termination = static_cast<Termination>(rep.termination);
  out.total_seconds = rep.total_seconds;
  out.free_dims = rep.free_dims;
  out.residual_dims = rep.residual_dims;
  out.active_factors = rep.active_factors;
  out.memory = {rep.memory.jacobian_bytes, rep.memory.preconditioner_bytes, rep.memory.workspace_bytes,
                rep.memory.graph_bytes};
  for (int i = 0; i < rep.iterations_run; ++i) {
    const gb_iteration_record& r = recs[static_cast<std::size_t>(i)];
    out.iterations.push_back({r.iteration, r.chi2_before, r.chi2_after, r.lambda, r.pcg_iterations,
                              r.pcg_converged != 0, r.pcg_relative_residual, r.low_quality_step != 0,
                              r.precond_fallback_blocks, r.accepted != 0, r.wall_seconds});
  }
  return out;
}

// ================================================================== BAL
namespace bal {

struct BALProblem {
  struct Observation {
    std::uint32_t camera_index;
    std::uint32_t point_index;
    double x;
    double y;
  };
  std::size_t num_cameras() const { return cameras.size(); }
  std::size_t num_points() const { return points.size(); }
  std::size_t num_observations() const { return observations.size(); }
  std::vector<Observation> observations;
  std::vector<std::array<double, 9>> cameras;
  std::vector<std::array<double, 3>> points;
};

template <typename FP, typename SP>
struct CameraTraits {
  static constexpr int dimension = 9;
  using Vertex = std::array<FP, 9>;
  static std::array<FP, 9> parameters(const Vertex& v) { return v; }
  static void update(Vertex& v, const FP* delta) {
    for (int i = 0; i < 9; ++i) v[i] += delta[i];
  }
  static void set_parameters(Vertex& v, const FP* block) {
    for (int i = 0; i < 9; ++i) v[i] = block[i];
  }
};

template <typename FP, typename SP>
struct Point3Traits {
  static constexpr int dimension = 3;
  using Vertex = std::array<FP, 3>;
  static std::array<FP, 3> parameters(const Vertex& v) { return v; }
  static void update(Vertex& v, const FP* delta) {
    for (int i = 0; i < 3; ++i) v[i] += delta[i];
  }
  static void set_parameters(Vertex& v, const FP* block) {
    for (int i = 0; i < 3; ++i) v[i] = block[i];
  }
};

template <typename FP, typename SP>
using CameraDescriptor = VertexDescriptor<FP, SP, CameraTraits<FP, SP>>;
template <typename FP, typename SP>
using Point3Descriptor = VertexDescriptor<FP, SP, Point3Traits<FP, SP>>;

template <typename FP, typename SP>
struct ReprojectionTraits {
  static constexpr int residual_dimension = 2;
  static constexpr bool kIsBalReprojection = true;
  using SlotDescriptors = std::tuple<CameraDescriptor<FP, SP>, Point3Descriptor<FP, SP>>;
  using Observation = std::array<FP, 2>;
  using ConstantData = std::uint8_t;
};

template <typename FP, typename SP>
using ReprojectionFactor = FactorDescriptor<FP, SP, ReprojectionTraits<FP, SP>>;

template <typename FP, typename SP>
struct BalGraph {
  std::vector<std::array<FP, 9>> cameras;
  std::vector<std::array<FP, 3>> points;
  std::unique_ptr<CameraDescriptor<FP, SP>> camera_desc;
  std::unique_ptr<Point3Descriptor<FP, SP>> point_desc;
  std::unique_ptr<ReprojectionFactor<FP, SP>> factor_desc;
  Graph<FP, SP> graph;
  std::size_t num_observations = 0;

  // BalGraph::mse (adapter.hpp:95-99), evaluated on the device.
  FP mse() {
    if (num_observations == 0) return FP(0);
    constexpr int prec = detail::precision_code<FP, SP>();
    std::vector<std::uint32_t> ci, pi;
    std::vector<FP> obs;
    std::vector<std::uint8_t> lvl;
    int lk;
    double d;
    factor_desc->export_bal(ci, pi, obs, lvl, lk, d);
    detail::Handle h;
    h.g = gb_create(prec, GB_ANALYTIC, graph.device());
    if (!h.g) detail::check(GB_ERR_NO_DEVICE);
    detail::check(gb_set_cameras(h.g, cameras.data(), cameras.size(), nullptr));
    detail::check(gb_set_points(h.g, points.data(), points.size(), nullptr));
    detail::check(gb_set_observations(h.g, ci.size(), ci.data(), pi.data(), obs.data(), nullptr, lk, d));
    double out = 0;
    detail::check(gb_mse(h.g, &out));
    return static_cast<FP>(out);
  }
};

// bal::build_graph (adapter.hpp:106-143)
template <typename FP, typename SP>
std::unique_ptr<BalGraph<FP, SP>> build_graph(const BALProblem& problem, DifferentiationMode mode,
                                              std::optional<double> huber_delta = std::nullopt) {
  auto bg = std::make_unique<BalGraph<FP, SP>>();
  bg->num_observations = problem.num_observations();
  bg->cameras.resize(problem.num_cameras());
  for (std::size_t c = 0; c < problem.num_cameras(); ++c)
    for (int k = 0; k < 9; ++k) bg->cameras[c][k] = static_cast<FP>(problem.cameras[c][k]);
  bg->points.resize(problem.num_points());
  for (std::size_t p = 0; p < problem.num_points(); ++p)
    for (int k = 0; k < 3; ++k) bg->points[p][k] = static_cast<FP>(problem.points[p][k]);
  bg->camera_desc = std::make_unique<CameraDescriptor<FP, SP>>();
  bg->camera_desc->reserve(bg->cameras.size());
  bg->graph.add_vertex_descriptor(bg->camera_desc.get());
  for (std::size_t c = 0; c < bg->cameras.size(); ++c) bg->camera_desc->add_vertex(c, &bg->cameras[c]);
  bg->point_desc = std::make_unique<Point3Descriptor<FP, SP>>();
  bg->point_desc->reserve(bg->points.size());
  bg->graph.add_vertex_descriptor(bg->point_desc.get());
  for (std::size_t p = 0; p < bg->points.size(); ++p) bg->point_desc->add_vertex(p, &bg->points[p]);
  bg->factor_desc = std::make_unique<ReprojectionFactor<FP, SP>>(bg->camera_desc.get(), bg->point_desc.get());
  bg->factor_desc->reserve(problem.num_observations());
  bg->factor_desc->set_differentiation_mode(mode);
  bg->graph.add_factor_descriptor(bg->factor_desc.get());
  const auto loss = huber_delta ? LossParams<FP>::Huber(static_cast<FP>(*huber_delta)) : LossParams<FP>::Default();
  for (const auto& obs : problem.observations)
    bg->factor_desc->add_factor({obs.camera_index, obs.point_index}, {static_cast<FP>(obs.x), static_cast<FP>(obs.y)},
                                nullptr, 0, loss);
  return bg;
}

}  // namespace bal
}  // namespace gopt
