// Host orchestration and the C ABI (include/gb_bal.h).
//
// One handle = one user graph (cameras, points, observations) bound to one
// CUDA device and one stream. gb_optimize uploads once, runs every LM
// iteration as a captured CUDA graph whose kernels read and write the
// device-resident State (no host decision inside an iteration), and writes
// the refined parameters back into the user's AoS buffers.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <thread>
#include <stdexcept>
#include <string>
#include <vector>

#include "activate.hpp"
#include "activate_dev.cuh"
#include "dist.hpp"
#include "gb_bal.h"
#include "kernels.cuh"
#include "hvp_pipe.cuh"
#include "hvp_rc.cuh"
#include "lin_seg.cuh"

namespace gb {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NoDevice : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define CK(x)                                                                                         \
  do {                                                                                                \
    cudaError_t err__ = (x);                                                                          \
    if (err__ != cudaSuccess)                                                                         \
      throw CudaError(std::string("CUDA error ") + cudaGetErrorString(err__) + " at " #x);            \
  } while (0)

// ------------------------------------------------------------ user graph data
struct GraphData {
  int precision = GB_FP64;
  int diff_mode = GB_ANALYTIC;
  int device = 0;
  void* cams = nullptr;
  void* pts = nullptr;
  uint64_t nc = 0, np = 0, ne = 0;
  std::vector<uint8_t> cam_fixed, pt_fixed;
  // Observation arrays are referenced, not copied (gb_set_observations): the
  // caller keeps them alive and unchanged until the next set or gb_destroy.
  const uint32_t* cam_idx = nullptr;
  const uint32_t* pt_idx = nullptr;
  const double* obs = nullptr;        // fp64 input as given, or obs_conv (fp32 input widened once)
  const uint8_t* level = nullptr;     // null: all level 0
  std::vector<double> obs_conv;
  int loss_kind = GB_LOSS_DEFAULT;
  double huber = 1.0;
  uint64_t revision = 1;
  int linear_solver = GB_SOLVER_PCG;
  std::shared_ptr<Reducer> reducer;  // null: single GPU
  int world() const { return reducer ? reducer->world() : 1; }
  int rank() const { return reducer ? reducer->rank() : 0; }
};

class SolverBase {
 public:
  virtual ~SolverBase() = default;
  virtual void optimize(const gb_lm_config& cfg, gb_solve_report* rep, gb_iteration_record* recs, int max_recs) = 0;
  virtual void begin(const gb_lm_config& cfg, gb_solve_report* rep) = 0;
  virtual void step(int n) = 0;
  virtual void end(gb_solve_report* rep, gb_iteration_record* recs, int max_recs) = 0;
  virtual void* stream() = 0;
  virtual void time_hvp(int reps, double* ms_pair, double* ms_tiles) = 0;
  virtual void hvp_bytes(double* kernel_bytes, double* reference_bytes) = 0;
  virtual void hvp_info(int32_t* path, double* algorithmic_bytes, double* algorithmic_flops) = 0;
  virtual int iteration_kernels() const = 0;  // kernel nodes of one captured LM iteration (0: not captured)
  virtual double residual_sum(int level, bool raw) = 0;
  virtual void ls_linearize(int level, double cmin, double cmax, int damping, double* chi2, int64_t* n, void* b,
                            void* diag, void* clamped, void* scaling, int32_t* finite) = 0;
  virtual void ls_hvp(const void* v, void* out, double lambda) = 0;
  virtual void ls_precond(double lambda, void* blocks, int32_t* fallbacks) = 0;
  virtual void ls_solve_step(double lambda, const gb_pcg_config& pcg, void* dx, gb_pcg_stats* st, double* pred,
                             int32_t* finite) = 0;
  virtual void ls_jacobians(void* out) = 0;
  virtual const Activation& activation() = 0;
  virtual std::string selfcheck(int level) = 0;
};

// ------------------------------------------------------------- device memory
// Process-wide cache of freed device blocks (>= 1 MiB), per device, so that a
// graph built after another one (bench e2e, repeated solves, tests) reuses its
// memory instead of paying cudaMalloc's page mapping again. Blocks are reused
// when they are at most 2x the request; the cache holds at most 1/3 of the
// device's memory and is flushed before an allocation is retried on OOM.
class BlockCache {
 public:
  static BlockCache& get() {
    static BlockCache c;
    return c;
  }
  // a cached block of at least `bytes` (at most 2x); *cap = its true size
  void* take(int dev, size_t bytes, size_t* cap) {
    std::lock_guard<std::mutex> lk(m_);
    auto& f = free_[dev];
    auto it = f.lower_bound(bytes);
    if (it == f.end() || it->first > 2 * bytes) return nullptr;
    void* p = it->second;
    *cap = it->first;
    held_[dev] -= it->first;
    f.erase(it);
    return p;
  }
  // returns false when the caller should cudaFree the block itself
  bool give(int dev, void* p, size_t bytes) {
    if (bytes < (1u << 20)) return false;
    std::lock_guard<std::mutex> lk(m_);
    size_t& total = total_[dev];
    if (!total) {  // the memory size of `dev` (not of the current device), queried once
      cudaDeviceProp prop;
      if (cudaGetDeviceProperties(&prop, dev) == cudaSuccess) total = prop.totalGlobalMem;
      if (!total) return false;
    }
    if (held_[dev] + bytes > total / 3) return false;
    free_[dev].emplace(bytes, p);
    held_[dev] += bytes;
    return true;
  }
  void flush(int dev) {
    std::lock_guard<std::mutex> lk(m_);
    for (auto& kv : free_[dev]) cudaFree(kv.second);
    free_[dev].clear();
    held_[dev] = 0;
  }

 private:
  std::mutex m_;
  std::map<int, std::multimap<size_t, void*>> free_;
  std::map<int, size_t> held_;
  std::map<int, size_t> total_;
};

// Page-locked host blocks for graph-owned parameter arrays (gb_host_alloc):
// uploads and write-backs from them run at full PCIe/C2C rate. Freed blocks
// are kept for the next graph (reuse when at most 2x the request, at most
// 8 GiB held), like the device BlockCache above.
class HostCache {
 public:
  static HostCache& get() {
    static HostCache c;
    return c;
  }
  void* alloc(size_t bytes) {
    if (!bytes) bytes = 1;
    {
      std::lock_guard<std::mutex> lk(m_);
      auto it = free_.lower_bound(bytes);
      if (it != free_.end() && it->first <= 2 * bytes) {
        void* p = it->second;
        held_ -= it->first;
        size_[p] = it->first;
        free_.erase(it);
        return p;
      }
    }
    void* p = nullptr;
    if (cudaHostAlloc(&p, bytes, cudaHostAllocPortable) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    std::lock_guard<std::mutex> lk(m_);
    size_[p] = bytes;
    return p;
  }
  void release(void* p) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(m_);
    auto it = size_.find(p);
    if (it == size_.end()) return;
    const size_t bytes = it->second;
    size_.erase(it);
    if (held_ + bytes > (size_t(8) << 30)) {
      cudaFreeHost(p);
      return;
    }
    free_.emplace(bytes, p);
    held_ += bytes;
  }

 private:
  std::mutex m_;
  std::multimap<size_t, void*> free_;
  std::map<void*, size_t> size_;
  size_t held_ = 0;
};

class DBuf {
 public:
  static constexpr size_t kSlack = 64;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { release(); }
  void release() {
    if (p_) {
      // stream work that may still use the block completes first (cudaFree's own
      // semantics), on the block's own device (another graph may have made a
      // different device current on this thread)
      int cur = -1;
      cudaGetDevice(&cur);
      if (cur != dev_) cudaSetDevice(dev_);
      cudaDeviceSynchronize();
      if (!BlockCache::get().give(dev_, p_, cap_)) cudaFree(p_);
      if (cur != dev_ && cur >= 0) cudaSetDevice(cur);
    }
    p_ = nullptr;
    bytes_ = cap_ = 0;
  }
  void* alloc(size_t bytes) {
    if (p_ && bytes + kSlack <= cap_) {  // the block already holds it
      bytes_ = bytes;
      return p_;
    }
    release();
    CK(cudaGetDevice(&dev_));
    const size_t want = bytes + kSlack;  // slack: 16-byte-widened bulk copies may read past the end
    size_t got = 0;
    void* c = BlockCache::get().take(dev_, want, &got);
    if (c) {
      p_ = c;
      cap_ = got;  // the block's true size (it goes back to the cache as such)
    } else {
      if (std::getenv("GB_TIMING") && want >= (1u << 20))
        std::fprintf(stderr, "[gb]   cudaMalloc %.1f MB (cache miss)\n", want / 1048576.0);
      cudaError_t e = cudaMalloc(&p_, want);
      if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        BlockCache::get().flush(dev_);
        e = cudaMalloc(&p_, want);
      }
      CK(e);
      cap_ = want;
    }
    bytes_ = bytes;
    return p_;
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p_);
  }
  size_t capacity() const { return cap_; }

 private:
  void* p_ = nullptr;
  size_t bytes_ = 0, cap_ = 0;
  int dev_ = 0;
};

template <typename T>
T* upload(DBuf& buf, const std::vector<T>& v, cudaStream_t s) {
  T* p = static_cast<T*>(buf.alloc(v.size() * sizeof(T)));
  if (!v.empty()) CK(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s));
  return p;
}

inline unsigned div_up(uint64_t a, uint64_t b) { return static_cast<unsigned>((a + b - 1) / b); }

// Setup phase timer: GB_TIMING=1 prints "[gb] phase ms" lines to stderr
// (synchronizing the stream at each mark, so only for diagnosis).
struct PhaseTimer {
  using Clock = std::chrono::steady_clock;
  bool on = false;
  cudaStream_t s = nullptr;
  Clock::time_point t;
  explicit PhaseTimer(cudaStream_t st) : s(st) {
    const char* e = std::getenv("GB_TIMING");
    on = e && *e && *e != '0';
    t = Clock::now();
  }
  void mark(const char* what) {
    if (!on) return;
    cudaStreamSynchronize(s);
    const auto n = Clock::now();
    std::fprintf(stderr, "[gb] %-28s %9.3f ms\n", what, std::chrono::duration<double, std::milli>(n - t).count());
    t = n;
  }
};

// --------------------------------------------------------------------- solver
template <typename FP, typename SP>
class Solver final : public SolverBase {
  using A = arith_t<SP>;
  using Clock = std::chrono::steady_clock;

 public:
  explicit Solver(GraphData& g) : g_(g) {
    CK(cudaSetDevice(g_.device));
    if (const char* e = std::getenv("GB_HVP_MINB")) hvp_minb_ = std::atoi(e);
    {
      int sms = 0, per = 0;
      CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g_.device));
      sms_ = static_cast<uint32_t>(sms);
      int o3 = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o3, k_precond_pts<FP, SP>, 256, 0));
      pt_occ_ = static_cast<unsigned>(std::max(1, o3));
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o3, k_chi2_tiles<FP, SP, false>, kTileThreads, 0));
      chi2_occ_ = static_cast<unsigned>(std::max(1, o3));
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_pcg_step<FP, SP>, 256, 0));
      coop_grid_ = static_cast<unsigned>(std::max(1, sms * std::max(1, per)));
      if (const char* e = std::getenv("GB_PCG_FUSED")) fused_pcg_ = std::atoi(e) != 0;
    }
    CK(cudaFuncSetAttribute(k_lin_normal<FP, SP, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(lin_normal_smem<FP>())));
    CK(cudaFuncSetAttribute(k_lin_normal<FP, SP, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(lin_normal_smem<FP>())));
    CK(cudaFuncSetAttribute(k_lin_normal<FP, SP, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(lin_normal_smem<FP>())));
    CK(cudaStreamCreateWithFlags(&s_, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s_up_, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&ev_up_, cudaEventDisableTiming));
    st_ = static_cast<State<FP>*>(st_buf_.alloc(sizeof(State<FP>)));
    CK(cudaMemsetAsync(st_, 0, sizeof(State<FP>), s_));
  }
  ~Solver() override {
    cudaSetDevice(g_.device);  // this handle's streams, events and blocks live there
    for (const auto& kv : phase_ms_)
      std::fprintf(stderr, "[gb phases] %-24s %8.3f ms x %d\n", kv.first.c_str(),
                   kv.second.first / std::max(1, kv.second.second), kv.second.second);
    if (rc_.prof) {  // GB_RC_DBG & 8: per-role mbarrier wait cycles of k_hvp_rc (summed over CTAs and launches)
      unsigned long long h[16] = {};
      if (cudaMemcpy(h, rc_.prof, sizeof(h), cudaMemcpyDeviceToHost) == cudaSuccess)
        std::fprintf(stderr,
                     "[rc prof] per-warp busy fractions: consumer wait ready %.3f | producer wait empty %.3f, "
                     "ring+setup %.3f, issue %.3f | preparer wait full %.3f\n",
                     double(h[0]) / h[7], 8.0 * h[2] / h[7], 8.0 * h[4] / h[7], 8.0 * h[5] / h[7], 8.0 * h[3] / h[7]);
      std::fprintf(stderr, "[rc prof] consumer wait work buffer %.3f | epilogue wait work %.3f\n",
                   double(h[1]) / h[7], 8.0 / 5.0 * h[6] / h[7]);
    }
    for (auto& e : ev_) cudaEventDestroy(e);
    if (graph_exec_) cudaGraphExecDestroy(graph_exec_);
    if (flag_host_) cudaFreeHost(flag_host_);
    cudaStreamDestroy(s_);
    cudaEventDestroy(ev_up_);
    cudaStreamDestroy(s_up_);
  }

  // current activation (the last level used; level 0 if never activated)
  const Activation& activation() override {
    ensure_structure(have_act_ ? act_level_ : 0);
    ensure_host_plan();
    return act_;
  }

  // device activation == host activation, array by array (empty string = ok)
  std::string selfcheck(int level) override {
    CK(cudaSetDevice(g_.device));
    have_act_ = false;
    ensure_structure(level);
    // host reference: the full activation, sliced to this rank when sharded
    Activation h;
    {
      Activation full;
      activate(activation_input(level), full);
      shard(full, g_.world(), g_.rank(), h);
    }
    std::string err;
    auto cmp = [&](const char* name, const auto* dptr, const auto& hv) {
      using T = typename std::decay_t<decltype(hv)>::value_type;
      std::vector<T> got(hv.size());
      if (!hv.empty()) CK(cudaMemcpy(got.data(), dptr, hv.size() * sizeof(T), cudaMemcpyDeviceToHost));
      if (got != hv && err.empty()) err = std::string("mismatch in ") + name;
    };
    if (h.ntiles != act_.ntiles || h.n_slots != act_.n_slots || h.nparts != act_.nparts || h.nchunks != act_.nchunks ||
        h.n_active != act_.n_active)
      return "count mismatch";
    if (h.tile_ebeg != act_.tile_ebeg || h.tile_pbeg != act_.tile_pbeg || h.tile_ecnt != act_.tile_ecnt ||
        h.tile_chunk_base != act_.tile_chunk_base || h.normal_tiles != act_.normal_tiles ||
        h.heavy_tiles != act_.heavy_tiles || h.tile_cam_off != act_.tile_cam_off)
      return "tile plan mismatch";
    cmp("pt_order", pt_order_dev_, h.pt_order);
    cmp("d_a", b_da_.as<uint32_t>(), h.d_a);
    cmp("d_cam", dev_.d_cam, h.d_cam);
    cmp("d_lpt", dev_.d_lpt, h.d_lpt);
    cmp("d_lcam", dev_.d_lcam, h.d_lcam);
    cmp("tile_cams", dev_.tile_cams, h.tile_cams);
    cmp("chunk_part_base", dev_.chunk_part_base, h.chunk_part_base);
    cmp("pt_slot_off", dev_.pt_slot_off, h.pt_slot_off);
    cmp("pt_slots", dev_.pt_slots, h.pt_slots);
    cmp("cam_part_off", dev_.cam_part_off, h.cam_part_off);
    cmp("cam_part_idx", dev_.cam_part_idx, h.cam_part_idx);
    return err;
  }

  // ---------------------------------------------------------------- optimize
  // levenberg_marquardt (levenberg_marquardt.hpp:115-224) in three phases.
  void begin(const gb_lm_config& cfg, gb_solve_report* rep) override {
    if (in_solve_) end(nullptr, nullptr, 0);
    t0_ = Clock::now();
    CK(cudaSetDevice(g_.device));
    PhaseTimer pt(s_);
    ensure_structure(cfg.level);
    pt.mark("begin: structure");
    upload_params();
    pt.mark("begin: upload params");
    cfg_ = cfg;
    State<FP> hs{};
    fill_config(hs, cfg);
    CK(cudaMemcpyAsync(st_, &hs, sizeof(hs), cudaMemcpyHostToDevice, s_));
    rec_buf_.alloc(sizeof(gb_iteration_record) * std::max(1, cfg.max_iterations));
    dev_.recs = rec_buf_.as<gb_iteration_record>();
    enqueue_linearize(1);
    CK(cudaMemcpyAsync(&hs, st_, sizeof(hs), cudaMemcpyDeviceToHost, s_));
    CK(cudaStreamSynchronize(s_));
    pt.mark("begin: initial linearize");
    const FP chi2 = hs.lin_chi2;
    if (!std::isfinite(static_cast<double>(chi2)))
      throw std::runtime_error("levenberg_marquardt: non-finite chi^2 at the initial parameters");
    gb_solve_report& r = rep_;
    r = gb_solve_report{};
    r.initial_chi2 = r.final_chi2 = static_cast<double>(chi2);
    r.free_dims = act_.free_dims;
    r.residual_dims = static_cast<int64_t>(2 * act_.n_active);
    r.active_factors = act_.n_active;
    r.memory = memory_account();
    r.termination = GB_TERM_MAX_ITERATIONS;
    r.h2d_bytes = static_cast<double>(h2d_bytes_);
    h2d_bytes_ = 0;
    launched_ = 0;
    max_it_ = 0;
    if (act_.free_dims == 0) {
      r.termination = GB_TERM_NO_FREE_PARAMETERS;
    } else if (cfg.max_iterations > 0) {
      // chi2, lambda0 = tau * max(D^2 clamped) (linear_system.hpp:94-99), nu = 2
      hs.chi2 = chi2;
      hs.lm_it = 0;
      hs.terminated = 0;
      hs.accepted_steps = 0;
      CK(cudaMemcpyAsync(st_, &hs, sizeof(hs), cudaMemcpyHostToDevice, s_));
      k_init_damping<FP, SP><<<col_grid(), 256, 0, s_>>>(dev_);
      CK(cudaGetLastError());
      if (dist()) {
        allreduce(dev_.redmax + kRedMaxDamp, 1, true);
        allreduce(red_s() + kRedDampAny, 1);
        fin(0);
      }
      pcg_max_it_ = cfg.pcg.max_iterations;
      if ((!dist() || g_.reducer->capturable()) && !phases_on_) {
        build_iteration_graph(cfg.pcg.max_iterations);
      } else if (graph_exec_) {
        cudaGraphExecDestroy(graph_exec_);
        graph_exec_ = nullptr;
      }
      max_it_ = cfg.max_iterations;
      ev_.resize(max_it_ + 1);
      for (auto& e : ev_) CK(cudaEventCreate(&e));
      CK(cudaStreamSynchronize(s_));
      pt.mark("begin: damping + graph capture");
    }
    r.setup_seconds = std::chrono::duration<double>(Clock::now() - t0_).count();
    in_solve_ = true;
    if (rep) *rep = r;
  }

  void step(int n) override {
    if (!in_solve_) throw std::logic_error("gb_step outside gb_begin/gb_end");
    for (int k = 0; k < n && launched_ < max_it_; ++k) {
      if (launched_ == 0) CK(cudaEventRecord(ev_[0], s_));
      if (graph_exec_)
        CK(cudaGraphLaunch(graph_exec_, s_));
      else
        enqueue_iteration(pcg_max_it_);
      ++launched_;
      CK(cudaEventRecord(ev_[launched_], s_));
    }
  }

  void end(gb_solve_report* rep, gb_iteration_record* recs, int max_recs) override {
    if (!in_solve_) throw std::logic_error("gb_end without gb_begin");
    in_solve_ = false;
    phase_flush();
    gb_solve_report& r = rep_;
    if (max_it_ > 0) {
      State<FP> hs;
      CK(cudaMemcpyAsync(&hs, st_, sizeof(hs), cudaMemcpyDeviceToHost, s_));
      CK(cudaStreamSynchronize(s_));
      const int nrec = hs.lm_it;
      std::vector<gb_iteration_record> hr(std::max(nrec, 1));
      if (nrec) CK(cudaMemcpy(hr.data(), dev_.recs, sizeof(gb_iteration_record) * nrec, cudaMemcpyDeviceToHost));
      for (int i = 0; i < nrec && i < launched_; ++i) {
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, ev_[i], ev_[i + 1]));
        hr[i].wall_seconds = ms * 1e-3;
      }
      for (auto& e : ev_) cudaEventDestroy(e);
      ev_.clear();
      r.termination = hs.terminated ? hs.termination : GB_TERM_MAX_ITERATIONS;
      r.accepted_steps = hs.accepted_steps;
      r.final_chi2 = static_cast<double>(hs.chi2);
      r.iterations_run = nrec;
      if (recs)
        for (int i = 0; i < std::min(nrec, max_recs); ++i) recs[i] = hr[i];
      download_params();
    }
    r.d2h_bytes = static_cast<double>(d2h_bytes_);
    d2h_bytes_ = 0;
    r.total_seconds = std::chrono::duration<double>(Clock::now() - t0_).count();
    if (rep) *rep = r;
  }

  void* stream() override { return s_; }

  void optimize(const gb_lm_config& cfg, gb_solve_report* rep, gb_iteration_record* recs, int max_recs) override {
    begin(cfg, nullptr);
    if (max_it_ > 0) {
      if (!flag_host_) CK(cudaHostAlloc(reinterpret_cast<void**>(&flag_host_), 64 * sizeof(int), cudaHostAllocDefault));
      std::vector<cudaEvent_t> flag_ev(max_it_);
      for (auto& e : flag_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      for (int it = 0; it < max_it_; ++it) {
        step(1);
        CK(cudaMemcpyAsync(&flag_host_[it % 64], &st_->terminated, sizeof(int), cudaMemcpyDeviceToHost, s_));
        CK(cudaEventRecord(flag_ev[it], s_));
        // look one iteration behind so the device always has queued work
        if (it >= 1) {
          CK(cudaEventSynchronize(flag_ev[it - 1]));
          if (flag_host_[(it - 1) % 64]) break;
        }
      }
      for (auto& e : flag_ev) cudaEventDestroy(e);
    }
    end(rep, recs, max_recs);
  }

  // Average device time of the HVP kernel pair (and of the tile kernel alone)
  // at the current linearization; the device State is saved and restored.
  // Bytes one HVP (as timed by time_hvp: tile pass + camera pass) must move
  // on the configured path, and the SURVEY.md §8(d) reference-layout figure
  // E (24 s_J + 8) + N (s_V + s_A) for comparison.
  void hvp_bytes(double* kernel_bytes, double* reference_bytes) override {
    if (!have_act_) throw std::logic_error("gb_hvp_bytes before any solve");
    const double sJ = sizeof(SP), sV = sizeof(SP), sA = sizeof(A), sF = sizeof(FP);
    const double E = static_cast<double>(act_.n_active), ns = static_cast<double>(act_.n_slots);
    const double N = static_cast<double>(act_.free_dims);
    const double np3 = 3.0 * act_.np, nc9 = 9.0 * act_.nc, nparts = static_cast<double>(act_.nparts);
    if (reference_bytes) *reference_bytes = E * (24 * sJ + 8) + N * (sV + sA);
    double b = 0;
    const Dev<FP, SP>& d = dev_;
    if (rc_ok_) {  // recompute HVP: tile blobs, X / p / z in, ap / p out, camera records and 15-value partials
      double aux = 0, lin = 0;
      for (uint32_t t : act_.normal_tiles) {
        const uint32_t ne = act_.tile_ecnt[t], npt = act_.tile_pbeg[t + 1] - act_.tile_pbeg[t];
        const uint32_t ncam = act_.tile_cam_off[t + 1] - act_.tile_cam_off[t];
        aux += aux_sections(ne, npt).bytes;
        lin += rc_lin_sections<FP>(ne, npt, ncam, d.w != nullptr).bytes;
      }
      b += aux + lin + np3 * 2 * sV + np3 * 2 * sV;              // blobs (incl. X); p, z in; ap, p out
      b += d.ntcams * (kRcRec * sF * 3.0 + 8.0);                 // camera record gathers, partials (write, read)
      b += act_.nc * kRcRec * sF * 2 + nc9 * (sF + sF + 2 * sV);  // camera records; x, cpre, p, z
      b += nc9 * (sV + sF + sV);                                 // camera p, D in; ap out
      if (kernel_bytes) *kernel_bytes = b;
      return;
    }
    if (pipe_ok_) {
      double aux = 0, lin = 0;
      for (uint32_t t : act_.normal_tiles) {
        const uint32_t ne = act_.tile_ecnt[t], npt = act_.tile_pbeg[t + 1] - act_.tile_pbeg[t];
        const uint32_t ncam = act_.tile_cam_off[t + 1] - act_.tile_cam_off[t];
        aux += aux_sections(ne, npt).bytes;
        lin += lin_sections<FP>(ne, npt, ncam, d.jfact != 0, d.w != nullptr).bytes;
      }
      const double rows = d.jfact ? kJFactRows : 24;
      b += jstore_elems<SP>(act_.n_slots, static_cast<int>(rows)) * sJ + aux + lin;  // J blocks, tile blobs
      b += np3 * (sV + sV);                            // p in, ap out
      b += d.ntcams * (cam_stride<A>() * sA * 2 + 4.0);  // tcv gather (tile_cams, write) + tile read
      b += 8.0 * nparts;                               // camera-run spans + storage slots
    } else {
      b += (d.J ? jstore_elems<SP>(act_.n_slots, 24) * sJ : 0) + ns * (4 + 2);  // J, camera and point indices
      b += np3 * (sA + sV + sF + sV + 1);              // vt, p, D in; ap out; free mask
      b += act_.np * 4.0 + ns * 2;                     // point slot lists
    }
    b += nparts * 9 * sF * 2 + nparts * 4;             // camera partial slots: write, read (+ index)
    b += nc9 * (sV + sF + sV);                         // camera p, D in; ap out
    if (kernel_bytes) *kernel_bytes = b;
  }

  void hvp_info(int32_t* path, double* algorithmic_bytes, double* algorithmic_flops) override {
    if (!have_act_) throw std::logic_error("gb_hvp_info before any solve");
    const double E = static_cast<double>(act_.n_active), N = static_cast<double>(act_.free_dims);
    const double sJ = sizeof(SP), sV = sizeof(SP), sA = sizeof(A), sF = sizeof(FP);
    const bool recompute = rc_ok_ || !dev_.J;
    if (path) *path = rc_ok_ ? 3 : (!dev_.J ? 0 : (pipe_ok_ ? 2 : 1));
    if (algorithmic_bytes)
      *algorithmic_bytes = recompute ? E * (2 * sF + 8) + static_cast<double>(ncols_) * sF + N * (sV + sA)
                                     : E * (24 * sJ + 8) + N * (sV + sA);
    if (algorithmic_flops) *algorithmic_flops = recompute ? E * 500.0 : 0.0;
  }

  int iteration_kernels() const override { return graph_exec_ ? graph_kernels_ : 0; }

  void time_hvp(int reps, double* ms_pair, double* ms_tiles) override {
    if (in_solve_) throw std::logic_error("gb_time_hvp during a solve");
    if (!have_act_) throw std::logic_error("gb_time_hvp before any solve");
    State<FP> saved;
    CK(cudaMemcpyAsync(&saved, st_, sizeof(saved), cudaMemcpyDeviceToHost, s_));
    CK(cudaStreamSynchronize(s_));
    State<FP> hs = saved;
    hs.iter_active = 1;
    hs.pcg_done = 0;
    CK(cudaMemcpyAsync(st_, &hs, sizeof(hs), cudaMemcpyHostToDevice, s_));
    cudaEvent_t a, b, c;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    CK(cudaEventCreate(&c));
    launch_hvp(dev_);  // warm
    CK(cudaEventRecord(a, s_));
    for (int i = 0; i < reps; ++i) launch_hvp(dev_);
    CK(cudaEventRecord(b, s_));
    for (int i = 0; i < reps; ++i) launch_hvp_tiles(dev_);
    CK(cudaEventRecord(c, s_));
    CK(cudaEventSynchronize(c));
    float m1 = 0, m2 = 0;
    CK(cudaEventElapsedTime(&m1, a, b));
    CK(cudaEventElapsedTime(&m2, b, c));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaEventDestroy(c);
    CK(cudaMemcpyAsync(st_, &saved, sizeof(saved), cudaMemcpyHostToDevice, s_));
    CK(cudaStreamSynchronize(s_));
    if (ms_pair) *ms_pair = m1 / reps;
    if (ms_tiles) *ms_tiles = m2 / reps;
  }

  double residual_sum(int level, bool raw) override {
    CK(cudaSetDevice(g_.device));
    ensure_structure(level);
    upload_params();
    k_cam_pre<FP, SP><<<std::max(1u, div_up(act_.nc, 128)), 128, 0, s_>>>(dev_, dev_.x, dev_.cpre_new, 2, 1);
    if (raw)
      k_chi2_tiles<FP, SP, true><<<chi2_grid(), kTileThreads, 0, s_>>>(dev_, dev_.x, 1);
    else
      k_chi2_tiles<FP, SP, false><<<chi2_grid(), kTileThreads, 0, s_>>>(dev_, dev_.x, 1);
    CK(cudaGetLastError());
    if (dist()) allreduce(&st_->chi2_new, 1);
    State<FP> hs;
    CK(cudaMemcpyAsync(&hs, st_, sizeof(hs), cudaMemcpyDeviceToHost, s_));
    CK(cudaStreamSynchronize(s_));
    return static_cast<double>(hs.chi2_new);
  }

  // ------------------------------------------------ LinearSystem debug surface
  void ls_linearize(int level, double cmin, double cmax, int damping, double* chi2, int64_t* n, void* b, void* diag,
                    void* clamped, void* scaling, int32_t* finite) override {
    CK(cudaSetDevice(g_.device));
    need_single();
    ensure_structure(level);
    ensure_host_plan();
    upload_params();
    gb_lm_config cfg;
    gb_default_config(&cfg);
    cfg.clamp_min = cmin;
    cfg.clamp_max = cmax;
    cfg.damping = damping;
    State<FP> hs{};
    fill_config(hs, cfg);
    CK(cudaMemcpyAsync(st_, &hs, sizeof(hs), cudaMemcpyHostToDevice, s_));
    enqueue_linearize(1);
    CK(cudaMemcpyAsync(&hs, st_, sizeof(hs), cudaMemcpyDeviceToHost, s_));
    CK(cudaStreamSynchronize(s_));
    ls_state_ = hs;
    ls_ready_ = true;
    if (chi2) *chi2 = static_cast<double>(hs.lin_chi2);
    if (n) *n = act_.free_dims;
    if (finite) *finite = hs.lin_finite;
    auto fetch = [&](const FP* src, void* dst) {
      if (!dst) return;
      std::vector<FP> h(ncols_);
      CK(cudaMemcpy(h.data(), src, ncols_ * sizeof(FP), cudaMemcpyDeviceToHost));
      FP* o = static_cast<FP*>(dst);
      for (size_t i = 0; i < ref_to_int_.size(); ++i) o[i] = h[ref_to_int_[i]];
    };
    fetch(dev_.b, b);
    fetch(dev_.clamped, clamped);
    fetch(dev_.D, scaling);
    if (diag) {
      std::vector<FP> hc(45ull * act_.nc), hp(6ull * act_.np);
      CK(cudaMemcpy(hc.data(), dev_.Hc, hc.size() * sizeof(FP), cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(hp.data(), dev_.Hp, hp.size() * sizeof(FP), cudaMemcpyDeviceToHost));
      FP* o = static_cast<FP*>(diag);
      for (uint64_t c = 0; c < act_.nc; ++c)
        if (act_.cam_col[c] >= 0)
          for (int k = 0; k < 9; ++k) o[act_.cam_col[c] + k] = hc[45 * c + p9(k, k)];
      for (uint64_t p = 0; p < act_.np; ++p)
        if (act_.pt_col[p] >= 0)
          for (int k = 0; k < 3; ++k) o[act_.pt_col[p] + k] = hp[6ull * act_.pt_rank[p] + p3(k, k)];
    }
  }

  void need_ls() const {
    if (!ls_ready_) throw std::logic_error("linear system not linearized (call gb_ls_linearize first)");
  }
  void need_single() const {
    if (g_.world() > 1) throw std::logic_error("the LinearSystem inspection surface needs world == 1");
  }

  void begin_solve_state(double lambda, const gb_pcg_config* pcg) {
    State<FP> hs = ls_state_;
    hs.iter_active = 1;
    hs.lambda_solve = static_cast<FP>(lambda);
    hs.lambda = static_cast<FP>(lambda);
    hs.pcg_done = hs.pcg_it = hs.pcg_conv = hs.pcg_zero = 0;
    hs.dir_pending = hs.x_pending = 0;
    hs.pcg_relres = 0;
    hs.fallbacks = 0;
    hs.schur = g_.linear_solver == GB_SOLVER_SCHUR ? 1 : 0;
    if (pcg) {
      hs.pcg_max_it = pcg->max_iterations;
      hs.pcg_tol = pcg->tolerance;
      hs.pcg_ratio = pcg->rejection_ratio;
      hs.normalize_rhs = pcg->normalize_rhs;
    }
    CK(cudaMemcpyAsync(st_, &hs, sizeof(hs), cudaMemcpyHostToDevice, s_));
  }

  void ls_hvp(const void* v, void* out, double lambda) override {
    need_ls();
    begin_solve_state(lambda, nullptr);
    std::vector<SP> hv(ncols_, narrow<SP>(0.0));
    const SP* vin = static_cast<const SP*>(v);
    for (size_t i = 0; i < ref_to_int_.size(); ++i) hv[ref_to_int_[i]] = vin[i];
    CK(cudaMemcpyAsync(dev_.p, hv.data(), ncols_ * sizeof(SP), cudaMemcpyHostToDevice, s_));
    k_make_vt<FP, SP><<<col_grid(), 256, 0, s_>>>(dev_);
    CK(cudaGetLastError());
    Dev<FP, SP> d = dev_;
    d.dbg_out = static_cast<A*>(dbg_buf_.alloc(ncols_ * sizeof(A)));
    launch_hvp(d);
    std::vector<A> h(ncols_);
    CK(cudaMemcpyAsync(h.data(), d.dbg_out, ncols_ * sizeof(A), cudaMemcpyDeviceToHost, s_));
    CK(cudaStreamSynchronize(s_));
    A* o = static_cast<A*>(out);
    for (size_t i = 0; i < ref_to_int_.size(); ++i) o[i] = h[ref_to_int_[i]];
  }

  void ls_precond(double lambda, void* blocks, int32_t* fallbacks) override {
    need_ls();
    begin_solve_state(lambda, nullptr);
    launch_precond();
    CK(cudaGetLastError());
    State<FP> hs;
    std::vector<FP> mc(45ull * act_.nc), mp(6ull * act_.np);
    CK(cudaMemcpyAsync(mc.data(), dev_.Mc, mc.size() * sizeof(FP), cudaMemcpyDeviceToHost, s_));
    CK(cudaMemcpyAsync(mp.data(), dev_.Mp, mp.size() * sizeof(FP), cudaMemcpyDeviceToHost, s_));
    CK(cudaMemcpyAsync(&hs, st_, sizeof(hs), cudaMemcpyDeviceToHost, s_));
    CK(cudaStreamSynchronize(s_));
    if (fallbacks) *fallbacks = hs.fallbacks;
    if (!blocks) return;
    FP* o = static_cast<FP*>(blocks);
    uint64_t base = 0;
    for (uint64_t c = 0; c < act_.nc; ++c) {
      if (act_.cam_col[c] < 0) continue;
      for (int i = 0; i < 9; ++i)
        for (int j = 0; j < 9; ++j) o[base + 9 * i + j] = mc[45 * c + p9(i, j)];
      base += 81;
    }
    for (uint64_t p = 0; p < act_.np; ++p) {
      if (act_.pt_col[p] < 0) continue;
      const uint64_t r = act_.pt_rank[p];
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) o[base + 3 * i + j] = mp[6 * r + p3(i, j)];
      base += 9;
    }
  }

  void ls_solve_step(double lambda, const gb_pcg_config& pcg, void* dx, gb_pcg_stats* stats, double* pred,
                     int32_t* finite) override {
    need_ls();
    begin_solve_state(lambda, &pcg);
    dev_.want_dx = 1;  // this surface returns dx; the LM loop's k_step skips the store
    enqueue_solve(pcg.max_iterations);
    dev_.want_dx = 0;
    State<FP> hs;
    CK(cudaMemcpyAsync(&hs, st_, sizeof(hs), cudaMemcpyDeviceToHost, s_));
    std::vector<FP> h(ncols_);
    CK(cudaMemcpyAsync(h.data(), dev_.dx, ncols_ * sizeof(FP), cudaMemcpyDeviceToHost, s_));
    CK(cudaStreamSynchronize(s_));
    if (dx) {
      FP* o = static_cast<FP*>(dx);
      for (size_t i = 0; i < ref_to_int_.size(); ++i) o[i] = h[ref_to_int_[i]];
    }
    if (stats) *stats = gb_pcg_stats{hs.pcg_it, hs.pcg_relres, hs.pcg_conv};
    if (pred) *pred = static_cast<double>(hs.pred);
    if (finite) *finite = hs.step_finite;
  }

  void ls_jacobians(void* out) override {
    need_ls();
    if (!dev_.J && (!rc_ok_ || g_.diff_mode == GB_DYNAMIC)) throw std::logic_error("dynamic mode stores no Jacobians");
    const uint64_t ns = act_.n_slots;
    std::vector<SP> h(24 * ns);
    {
      DBuf full;
      SP* fj = static_cast<SP*>(full.alloc(24 * ns * sizeof(SP)));
      if (dev_.J)
        k_expand_J<FP, SP><<<grid_for(ns), 256, 0, s_>>>(dev_, fj);
      else  // recompute path: the J a store would hold, from the linearize chain at x
        k_eval_J<FP, SP><<<act_.ntiles, 128, 0, s_>>>(dev_, fj);
      CK(cudaGetLastError());
      CK(cudaMemcpyAsync(h.data(), fj, h.size() * sizeof(SP), cudaMemcpyDeviceToHost, s_));
      CK(cudaStreamSynchronize(s_));
    }
    SP* o = static_cast<SP*>(out);
    for (uint64_t d = 0; d < ns; ++d) {
      if (act_.d_a[d] == kNoKey) continue;
      const uint64_t a = act_.d_a[d];
      for (int k = 0; k < 24; ++k) o[24 * a + k] = h[k * ns + d];
    }
  }

 private:
  // ------------------------------------------------------------ structure
  ActivationInput activation_input(int level) const {
    ActivationInput in;
    in.nc = g_.nc;
    in.np = g_.np;
    in.ne = g_.ne;
    in.cam = g_.cam_idx;
    in.pt = g_.pt_idx;
    in.level = g_.level;
    in.cam_fixed = g_.cam_fixed.empty() ? nullptr : g_.cam_fixed.data();
    in.pt_fixed = g_.pt_fixed.empty() ? nullptr : g_.pt_fixed.data();
    in.active_level = level;
    in.tile_edge_cap = tile_edge_cap();
    return in;
  }

  // Greedy tile edge budget (experiments: GB_TILE_CAP). Measured on the
  // recompute path at Final: 512 edges 0.739 ms per HVP, 480: 0.814, 448:
  // 0.858 — the per-tile costs outweigh the shorter segments.
  uint32_t tile_edge_cap() const {
    uint32_t cap = static_cast<uint32_t>(kTileEdges);
    if (const char* e = std::getenv("GB_TILE_CAP")) cap = static_cast<uint32_t>(std::atoi(e));
    return std::max<uint32_t>(32, std::min<uint32_t>(cap, kTileEdges));
  }

  void ensure_structure(int level) {
    pts_staged_ = false;  // set again only by a device activation run below
    if (have_act_ && act_rev_ == g_.revision && act_level_ == level) return;
    if (!g_.cams || !g_.pts) throw std::logic_error("cameras and points must be set before solving");
    host_plan_ = false;
    device_structure(level);  // sharded: this rank's point-tile range only
    have_act_ = true;
    act_rev_ = g_.revision;
    act_level_ = level;
    ls_ready_ = false;
    if (graph_exec_) {
      cudaGraphExecDestroy(graph_exec_);
      graph_exec_ = nullptr;
    }
    PhaseTimer pt(s_);
    allocate_work();
    pt.mark("allocate work");
  }

  // The host activation (activate.cpp) for the debug surface of a device-
  // activated graph: identical structures (gb_activation_selfcheck), plus the
  // reference column map and incidence CSRs.
  void ensure_host_plan() {
    if (host_plan_) return;
    need_single();
    activate(activation_input(act_level_), act_);
    host_plan_ = true;
    build_ref_map();
  }

  void build_ref_map() {
    const uint64_t nc = act_.nc, np = act_.np;
    ref_to_int_.assign(act_.free_dims, 0);
    for (uint64_t c = 0; c < nc; ++c)
      if (act_.cam_col[c] >= 0)
        for (int k = 0; k < 9; ++k) ref_to_int_[act_.cam_col[c] + k] = 9 * c + k;
    for (uint64_t i = 0; i < np; ++i) {
      const uint64_t p = act_.pt_order[i];
      if (act_.pt_col[p] >= 0)
        for (int k = 0; k < 3; ++k) ref_to_int_[act_.pt_col[p] + k] = 9 * nc + 3 * i + k;
    }
  }

  void set_counts() {
    Dev<FP, SP>& d = dev_;
    ncols_ = 9 * act_.nc + 3 * act_.np;
    d.nc = static_cast<uint32_t>(act_.nc);
    d.np = static_cast<uint32_t>(act_.np);
    d.na = static_cast<uint32_t>(act_.n_slots);
    d.ntiles = act_.ntiles;
    d.nparts = act_.nparts;
    d.ncols = ncols_;
  }

  // ---- host activation -> device arrays (sharded path)
  void upload_structure_host() {
    const uint64_t nc = act_.nc, np = act_.np, ns = act_.n_slots;
    dev_ = Dev<FP, SP>{};
    set_counts();
    Dev<FP, SP>& d = dev_;
    size_t h2d = 0;
    auto up = [&](DBuf& buf, const auto& v) {
      h2d += v.size() * sizeof(v[0]);
      return upload(buf, v, s_);
    };
    std::vector<uint8_t> col_free(ncols_, 0);
    for (uint64_t c = 0; c < nc; ++c)
      if (act_.cam_col[c] >= 0)
        for (int k = 0; k < 9; ++k) col_free[9 * c + k] = 1;
    for (uint64_t i = 0; i < np; ++i)  // local internal point i -> point id pt_order[i]
      if (act_.pt_col[act_.pt_order[i]] >= 0)
        for (int k = 0; k < 3; ++k) col_free[9 * nc + 3 * i + k] = 1;
    if (g_.world() == 1) build_ref_map();
    d.col_free = up(b_col_free_, col_free);
    d.d_cam = up(b_dcam_, act_.d_cam);
    d.d_lpt = up(b_dlpt_, act_.d_lpt);
    d.d_lcam = up(b_dlcam_, act_.d_lcam);
    std::vector<FP> obs(2 * ns, FP(0));
    for (uint64_t e = 0; e < ns; ++e) {
      if (act_.d_a[e] == kNoKey) continue;
      const uint64_t i = act_.active[act_.d_a[e]];
      obs[e] = static_cast<FP>(g_.obs[2 * i]);
      obs[ns + e] = static_cast<FP>(g_.obs[2 * i + 1]);
    }
    d.d_obs = up(b_obs_, obs);
    d.tile_ebeg = up(b_tile_ebeg_, act_.tile_ebeg);
    d.tile_ecnt = up(b_tile_ecnt_, act_.tile_ecnt);
    d.tile_cam_off = up(b_tile_cam_off_, act_.tile_cam_off);
    d.tile_cams = up(b_tile_cams_, act_.tile_cams);
    d.normal_tiles = up(b_normal_, act_.normal_tiles);
    d.heavy_tiles = up(b_heavy_, act_.heavy_tiles);
    d.n_normal = static_cast<uint32_t>(act_.normal_tiles.size());
    d.n_heavy = static_cast<uint32_t>(act_.heavy_tiles.size());
    d.tile_pbeg = up(b_tile_pbeg_, act_.tile_pbeg);
    d.tile_chunk_base = up(b_tile_chunk_, act_.tile_chunk_base);
    d.chunk_part_base = up(b_chunk_part_, act_.chunk_part_base);
    d.pt_slot_off = up(b_pt_slot_off_, act_.pt_slot_off);
    d.pt_slots = up(b_pt_slots_, act_.pt_slots);
    d.cam_part_off = up(b_cam_part_off_, act_.cam_part_off);
    d.cam_part_idx = up(b_cam_part_idx_, act_.cam_part_idx);
    pt_order_dev_ = up(b_pt_order_, act_.pt_order);
    h2d_bytes_ += h2d;
  }

  // ---- device activation (single GPU): activate_dev.cuh
  template <typename T>
  T* scratch(DBuf& b, uint64_t n) {
    return static_cast<T*>(b.alloc(std::max<uint64_t>(1, n) * sizeof(T)));
  }
  template <typename T>
  T* to_dev(DBuf& b, const std::vector<T>& v) {
    h2d_bytes_ += v.size() * sizeof(T);
    return upload(b, v, s_);
  }
  template <typename T>
  T* to_dev(DBuf& b, const T* p, uint64_t n) {
    h2d_bytes_ += n * sizeof(T);
    T* d = static_cast<T*>(b.alloc(std::max<uint64_t>(1, n) * sizeof(T)));
    if (n) CK(cudaMemcpyAsync(d, p, n * sizeof(T), cudaMemcpyHostToDevice, s_));
    return d;
  }
  // CUB temp storage: sized for the largest request seen so far with 2x
  // headroom, so activation's growing requests do not re-allocate (a
  // re-allocation synchronizes the device, stalling the overlapped uploads)
  void* cub_temp(size_t bytes) {
    if (b_cub_.as<void>() && bytes + DBuf::kSlack <= b_cub_.capacity()) return b_cub_.as<void>();
    return b_cub_.alloc(std::max<size_t>(bytes, 2 * b_cub_.capacity()) + (size_t(4) << 20));
  }
  void cub_scan_excl(const uint32_t* in, uint32_t* out, uint64_t n) {
    size_t tmp = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, static_cast<int64_t>(n), s_));
    CK(cub::DeviceScan::ExclusiveSum(cub_temp(tmp), tmp, in, out, static_cast<int64_t>(n), s_));
  }
  void cub_scan_incl(const uint32_t* in, uint32_t* out, uint64_t n) {
    size_t tmp = 0;
    CK(cub::DeviceScan::InclusiveSum(nullptr, tmp, in, out, static_cast<int64_t>(n), s_));
    CK(cub::DeviceScan::InclusiveSum(cub_temp(tmp), tmp, in, out, static_cast<int64_t>(n), s_));
  }
  template <typename K>
  void cub_sort(const K* kin, K* kout, const uint32_t* vin, uint32_t* vout, uint64_t n, int end_bit) {
    size_t tmp = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kin, kout, vin, vout, static_cast<int64_t>(n), 0, end_bit, s_));
    CK(cub::DeviceRadixSort::SortPairs(cub_temp(tmp), tmp, kin, kout, vin, vout, static_cast<int64_t>(n), 0,
                                       end_bit, s_));
  }
  unsigned grid_for(uint64_t n) const {
    return std::max(1u, std::min(div_up(n, 256), 148u * 16u));
  }

  void device_structure(int level) {
    using namespace actdev;
    const uint64_t nc = g_.nc, np = g_.np, ne = g_.ne;
    act_ = Activation();
    act_.nc = nc;
    act_.np = np;
    act_.level = level;
    // columns (vertex_descriptor.hpp:115-126) - host, O(nc + np)
    for (uint64_t c = 0; c < nc; ++c) act_.free_cams += (g_.cam_fixed.empty() || !g_.cam_fixed[c]) ? 1 : 0;
    for (uint64_t p = 0; p < np; ++p) act_.free_pts += (g_.pt_fixed.empty() || !g_.pt_fixed[p]) ? 1 : 0;
    act_.free_dims = 9 * act_.free_cams + 3 * act_.free_pts;

    PhaseTimer ptm(s_);
    DBuf s_cam, s_pt, s_lvl, s_cfix, s_pfix, s_obs, s_flag, s_pos, s_cam_a, s_pt_a, s_entry, s_key, s_key2, s_val, s_val2,
        s_rank, s_deg, s_degi, s_rb, s_k64, s_k64b, s_order, s_pkey, s_pval, s_pkey2, s_pval2, s_hc, s_hr, s_ic, s_ir,
        s_runcam, s_runcam2, s_slots, s_cnt, s_bad;
    const uint32_t* cam = to_dev(s_cam, g_.cam_idx, ne);
    const uint32_t* pt = to_dev(s_pt, g_.pt_idx, ne);
    const uint8_t* lvl = g_.level ? to_dev(s_lvl, g_.level, ne) : nullptr;
    const uint8_t* cfix = g_.cam_fixed.empty() ? nullptr : to_dev(s_cfix, g_.cam_fixed);
    const uint8_t* pfix = g_.pt_fixed.empty() ? nullptr : to_dev(s_pfix, g_.pt_fixed);
    // observations are first needed by k_place: their upload (2/3 of the
    // input bytes) runs on a side stream under compaction, point ordering and
    // the host tile pass
    double* obs = static_cast<double*>(s_obs.alloc(std::max<uint64_t>(1, 2 * ne) * sizeof(double)));
    if (ne) CK(cudaMemcpyAsync(obs, g_.obs, 2 * ne * sizeof(double), cudaMemcpyHostToDevice, s_up_));
    {  // the point parameters too (upload_params then only gathers them into the internal order)
      FP* stage = static_cast<FP*>(b_ptstage_.alloc(std::max<uint64_t>(1, 3 * np) * sizeof(FP)));
      if (np) CK(cudaMemcpyAsync(stage, g_.pts, 3 * np * sizeof(FP), cudaMemcpyHostToDevice, s_up_));
      pts_staged_ = true;
    }
    CK(cudaEventRecord(ev_up_, s_up_));
    h2d_bytes_ += 2 * ne * sizeof(double);
    ptm.mark("act: h2d edges");
    {  // CUB temp storage for the largest sort / scan of this activation, sized up
       // front: growing it later would synchronize the device mid-activation
      size_t t1 = 0, t2 = 0, t3 = 0;
      CK(cub::DeviceRadixSort::SortPairs(nullptr, t1, static_cast<const uint64_t*>(nullptr),
                                         static_cast<uint64_t*>(nullptr), static_cast<const uint32_t*>(nullptr),
                                         static_cast<uint32_t*>(nullptr), static_cast<int64_t>(ne), 0, 64, s_));
      CK(cub::DeviceRadixSort::SortPairs(nullptr, t2, static_cast<const uint32_t*>(nullptr),
                                         static_cast<uint32_t*>(nullptr), static_cast<const uint32_t*>(nullptr),
                                         static_cast<uint32_t*>(nullptr), static_cast<int64_t>(std::max(ne, np)), 0, 32,
                                         s_));
      CK(cub::DeviceScan::InclusiveSum(nullptr, t3, static_cast<const uint32_t*>(nullptr),
                                       static_cast<uint32_t*>(nullptr), static_cast<int64_t>(ne + np + 1), s_));
      cub_temp(std::max(t1, std::max(t2, t3)));
    }
    uint32_t* flag = scratch<uint32_t>(s_flag, ne + 1);
    uint32_t* pos = scratch<uint32_t>(s_pos, ne + 1);
    int* bad = scratch<int>(s_bad, 1);
    CK(cudaMemsetAsync(bad, 0, sizeof(int), s_));
    CK(cudaMemsetAsync(flag + ne, 0, sizeof(uint32_t), s_));
    k_flags<<<grid_for(ne), 256, 0, s_>>>(ne, cam, pt, lvl, level, static_cast<uint32_t>(nc), static_cast<uint32_t>(np),
                                          flag, bad);
    CK(cudaGetLastError());
    cub_scan_excl(flag, pos, ne + 1);
    uint32_t na32 = 0;
    int hbad = 0;
    CK(cudaMemcpyAsync(&na32, pos + ne, sizeof(uint32_t), cudaMemcpyDeviceToHost, s_));
    CK(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s_));
    CK(cudaStreamSynchronize(s_));
    ptm.mark("act:  flags + count");
    if (hbad) {  // reproduce the exact diagnostic (resolve_slots, factor_descriptor.hpp:549-558)
      Activation tmp;
      activate(activation_input(level), tmp);
    }
    const uint64_t na = na32;
    act_.n_active = na;
    uint32_t* cam_a = scratch<uint32_t>(s_cam_a, na);
    uint32_t* pt_a = scratch<uint32_t>(s_pt_a, na);
    uint32_t* entry_a = scratch<uint32_t>(s_entry, na);
    k_compact<<<grid_for(ne), 256, 0, s_>>>(ne, flag, pos, cam, pt, cam_a, pt_a, entry_a);
    ptm.mark("act:  compact");
    // internal point order: stable sort by smallest active camera
    uint32_t* key = scratch<uint32_t>(s_key, np);
    uint32_t* key2 = scratch<uint32_t>(s_key2, np);
    uint32_t* val = scratch<uint32_t>(s_val, np);
    uint32_t* deg = scratch<uint32_t>(s_deg, np);
    k_fill_u32<<<grid_for(np), 256, 0, s_>>>(np, static_cast<uint32_t>(nc), key);
    CK(cudaMemsetAsync(deg, 0, std::max<uint64_t>(1, np) * sizeof(uint32_t), s_));
    k_iota<<<grid_for(np), 256, 0, s_>>>(np, val);
    k_point_stats<<<grid_for(na), 256, 0, s_>>>(na, cam_a, pt_a, key, deg);
    CK(cudaGetLastError());
    ptm.mark("act:  point stats");
    uint32_t* pt_order = static_cast<uint32_t*>(b_pt_order_.alloc(std::max<uint64_t>(1, np) * sizeof(uint32_t)));
    cub_sort<uint32_t>(key, key2, val, pt_order, np, bits_for(nc + 1));
    pt_order_dev_ = pt_order;
    ptm.mark("act:  point sort");
    uint32_t* rank = scratch<uint32_t>(s_rank, np);
    uint32_t* degi = scratch<uint32_t>(s_degi, np + 1);
    CK(cudaMemsetAsync(degi + np, 0, sizeof(uint32_t), s_));
    k_rank<<<grid_for(np), 256, 0, s_>>>(np, pt_order, deg, rank, degi);
    CK(cudaGetLastError());
    // degrees to page-locked host memory (the host greedy pass reads them)
    struct HostBlock {
      void* p;
      ~HostBlock() { HostCache::get().release(p); }
    } hb{HostCache::get().alloc(std::max<uint64_t>(1, np) * sizeof(uint32_t))};
    std::vector<uint32_t> hdeg_fallback;
    uint32_t* hdeg = static_cast<uint32_t*>(hb.p);
    if (!hdeg) {
      hdeg_fallback.resize(np);
      hdeg = hdeg_fallback.data();
    }
    if (np) CK(cudaMemcpyAsync(hdeg, degi, np * sizeof(uint32_t), cudaMemcpyDeviceToHost, s_));
    CK(cudaStreamSynchronize(s_));
    // tiles: the host greedy over degrees (activate.cpp greedy_tiles), over ALL
    // points: the tile plan, and with it every rank's shard, is global
    ptm.mark("act: compact + point order");
    std::vector<uint32_t> gpbeg, greal;
    greedy_tiles(hdeg, np, gpbeg, greal, nullptr, tile_edge_cap());
    ptm.mark("act: host greedy tiles");
    const uint32_t GT = static_cast<uint32_t>(gpbeg.size() - 1);
    std::vector<uint32_t> gebeg(GT + 1, 0);
    {
      uint64_t slot = 0;
      for (uint32_t t = 0; t < GT; ++t) {
        gebeg[t] = static_cast<uint32_t>(slot);
        slot += (greal[t + 1] - greal[t] + kJBlock - 1) / kJBlock * kJBlock;
        if (slot > 0xffffffffull) throw std::invalid_argument("more than 2^32 padded edge slots");
      }
      gebeg[GT] = static_cast<uint32_t>(slot);
    }
    // this rank's contiguous tile range [t0, t1) / internal points [p0, p1)
    // (shard_bounds: the same balance as the host shard(); world 1: everything)
    uint32_t t0 = 0, t1 = GT, p0 = 0, p1 = static_cast<uint32_t>(np);
    if (g_.reducer) {
      const int W = g_.world();
      shard_p0_.assign(W + 1, 0);
      for (int r = 0; r < W; ++r) {
        uint32_t a0, a1, q0, q1;
        shard_bounds(gebeg.data(), gpbeg.data(), GT, W, r, &a0, &a1, &q0, &q1);
        shard_p0_[r] = q0;
        shard_p0_[r + 1] = q1;
      }
      shard_bounds(gebeg.data(), gpbeg.data(), GT, W, g_.rank(), &t0, &t1, &p0, &p1);
      full_np_ = np;  // the write-back scatters every rank's points through the global order
      full_pt_order_.resize(np);
      if (np) CK(cudaMemcpyAsync(full_pt_order_.data(), pt_order, np * sizeof(uint32_t), cudaMemcpyDeviceToHost, s_));
    }
    const uint32_t T = t1 - t0;
    const uint64_t npl = p1 - p0;
    act_.np = npl;
    act_.ntiles = T;
    act_.tile_pbeg.resize(T + 1);
    act_.tile_ecnt.resize(T);
    act_.tile_ebeg.assign(T + 1, 0);
    act_.tile_chunk_base.assign(T + 1, 0);
    std::vector<uint32_t> real_beg(T + 1);
    for (uint32_t t = 0; t <= T; ++t) {
      act_.tile_pbeg[t] = gpbeg[t0 + t] - p0;
      act_.tile_ebeg[t] = gebeg[t0 + t] - gebeg[t0];
      real_beg[t] = greal[t0 + t] - greal[t0];
    }
    for (uint32_t t = 0; t < T; ++t) {
      act_.tile_ecnt[t] = real_beg[t + 1] - real_beg[t];
      act_.tile_chunk_base[t + 1] = act_.tile_chunk_base[t] + (act_.tile_ecnt[t] + 31) / 32;
    }
    act_.n_slots = act_.tile_ebeg[T];
    act_.nchunks = act_.tile_chunk_base[T];
    const uint64_t ns = act_.n_slots;
    const uint64_t nal = real_beg[T];  // this rank's active edges
    dev_ = Dev<FP, SP>{};
    set_counts();
    Dev<FP, SP>& d = dev_;
    d.tile_pbeg = to_dev(b_tile_pbeg_, act_.tile_pbeg);
    d.tile_ebeg = to_dev(b_tile_ebeg_, act_.tile_ebeg);
    d.tile_ecnt = to_dev(b_tile_ecnt_, act_.tile_ecnt);
    d.tile_chunk_base = to_dev(b_tile_chunk_, act_.tile_chunk_base);
    const uint32_t* rb = to_dev(s_rb, real_beg);
    // device edge order: stable sort by (tile, camera) over factor order
    uint64_t* k64 = scratch<uint64_t>(s_k64, na);
    uint64_t* k64b = scratch<uint64_t>(s_k64b, na);
    uint32_t* vals = scratch<uint32_t>(s_val2, na);
    uint32_t* order = scratch<uint32_t>(s_order, na);
    k_edge_keys<<<grid_for(na), 256, 0, s_>>>(na, cam_a, pt_a, rank, d.tile_pbeg, T, p0, p1, k64, vals);
    CK(cudaGetLastError());
    // other ranks' edges carry the sentinel tile T: the first nal sorted keys are this rank's
    cub_sort<uint64_t>(k64, k64b, vals, order, na, 32 + bits_for(T));
    // padded slot arrays
    uint32_t* d_a = static_cast<uint32_t*>(b_da_.alloc(std::max<uint64_t>(1, ns) * sizeof(uint32_t)));
    uint32_t* d_cam = static_cast<uint32_t*>(b_dcam_.alloc(std::max<uint64_t>(1, ns) * sizeof(uint32_t)));
    uint16_t* d_lpt = static_cast<uint16_t*>(b_dlpt_.alloc(std::max<uint64_t>(1, ns) * sizeof(uint16_t)));
    uint16_t* d_lcam = static_cast<uint16_t*>(b_dlcam_.alloc(std::max<uint64_t>(1, ns) * sizeof(uint16_t)));
    FP* d_obs = static_cast<FP*>(b_obs_.alloc(std::max<uint64_t>(1, 2 * ns) * sizeof(FP)));
    CK(cudaMemsetAsync(d_a, 0xff, std::max<uint64_t>(1, ns) * sizeof(uint32_t), s_));
    CK(cudaMemsetAsync(d_lpt, 0, std::max<uint64_t>(1, ns) * sizeof(uint16_t), s_));
    CK(cudaMemsetAsync(d_obs, 0, std::max<uint64_t>(1, 2 * ns) * sizeof(FP), s_));
    uint32_t* pkey = scratch<uint32_t>(s_pkey, na);
    uint32_t* pval = scratch<uint32_t>(s_pval, na);
    uint32_t* hc = scratch<uint32_t>(s_hc, na);
    uint32_t* hr = scratch<uint32_t>(s_hr, na);
    CK(cudaStreamWaitEvent(s_, ev_up_, 0));  // observations uploaded
    k_place<FP><<<grid_for(nal), 256, 0, s_>>>(nal, k64b, order, cam_a, pt_a, entry_a, rank, p0, rb, d.tile_ebeg,
                                                d.tile_pbeg, obs, ns, d_a, d_cam, d_lpt, d_obs, pkey, pval, hc, hr);
    CK(cudaGetLastError());
    uint32_t* ic = scratch<uint32_t>(s_ic, na);
    uint32_t* ir = scratch<uint32_t>(s_ir, na);
    cub_scan_incl(hc, ic, nal);
    cub_scan_incl(hr, ir, nal);
    uint32_t* tile_cam_off = static_cast<uint32_t*>(b_tile_cam_off_.alloc((T + 1) * sizeof(uint32_t)));
    uint32_t* chunk_part_base =
        static_cast<uint32_t*>(b_chunk_part_.alloc((act_.nchunks + 1) * sizeof(uint32_t)));
    k_tile_offsets<<<grid_for(T + 1), 256, 0, s_>>>(T, nal, rb, d.tile_ecnt, d.tile_chunk_base, ic, ir, tile_cam_off,
                                                     chunk_part_base);
    CK(cudaGetLastError());
    act_.tile_cam_off.resize(T + 1);
    CK(cudaMemcpyAsync(act_.tile_cam_off.data(), tile_cam_off, (T + 1) * sizeof(uint32_t), cudaMemcpyDeviceToHost, s_));
    uint32_t nparts = 0;
    CK(cudaMemcpyAsync(&nparts, chunk_part_base + act_.nchunks, sizeof(uint32_t), cudaMemcpyDeviceToHost, s_));
    CK(cudaStreamSynchronize(s_));
    ptm.mark("act: edge sort + place");
    act_.nparts = nparts;
    d.nparts = nparts;
    const uint32_t ncams_total = act_.tile_cam_off[T];
    uint32_t* tile_cams = static_cast<uint32_t*>(b_tile_cams_.alloc(std::max<uint32_t>(1, ncams_total) * sizeof(uint32_t)));
    uint32_t* run_cam = scratch<uint32_t>(s_runcam, nparts);
    k_runs<<<grid_for(nal), 256, 0, s_>>>(nal, k64b, rb, d.tile_ebeg, tile_cam_off, hc, ic, hr, ir, d_lcam, tile_cams,
                                          run_cam);
    k_pad<<<grid_for(T), 256, 0, s_>>>(T, d.tile_ebeg, d.tile_ecnt, d_cam, d_lcam);
    CK(cudaGetLastError());
    // per-point slot lists: stable sort of (point rank, slot) + degree scan
    uint32_t* pkey2 = scratch<uint32_t>(s_pkey2, na);
    uint32_t* pval2 = scratch<uint32_t>(s_pval2, na);
    cub_sort<uint32_t>(pkey, pkey2, pval, pval2, nal, bits_for(npl));
    uint16_t* pt_slots = static_cast<uint16_t*>(b_pt_slots_.alloc(std::max<uint64_t>(1, nal) * sizeof(uint16_t)));
    k_u32_to_u16<<<grid_for(nal), 256, 0, s_>>>(nal, pval2, pt_slots);
    uint32_t* pt_slot_off = static_cast<uint32_t*>(b_pt_slot_off_.alloc((npl + 1) * sizeof(uint32_t)));
    cub_scan_excl(degi + p0, pt_slot_off, npl + 1);  // degi[p1] is never summed (exclusive)
    // camera -> partial-slot CSR
    uint32_t* slots = scratch<uint32_t>(s_slots, nparts);
    uint32_t* runcam2 = scratch<uint32_t>(s_runcam2, nparts);
    k_iota<<<grid_for(nparts), 256, 0, s_>>>(nparts, slots);
    uint32_t* cam_part_idx = static_cast<uint32_t*>(b_cam_part_idx_.alloc(std::max<uint32_t>(1, nparts) * sizeof(uint32_t)));
    cub_sort<uint32_t>(run_cam, runcam2, slots, cam_part_idx, nparts, bits_for(nc));
    uint32_t* cnt = scratch<uint32_t>(s_cnt, nc + 1);
    CK(cudaMemsetAsync(cnt, 0, (nc + 1) * sizeof(uint32_t), s_));
    k_hist<<<grid_for(nparts), 256, 0, s_>>>(nparts, run_cam, cnt);
    uint32_t* cam_part_off = static_cast<uint32_t*>(b_cam_part_off_.alloc((nc + 1) * sizeof(uint32_t)));
    cub_scan_excl(cnt, cam_part_off, nc + 1);
    // columns: free mask in internal order
    uint8_t* col_free = static_cast<uint8_t*>(b_col_free_.alloc(std::max<uint64_t>(1, ncols_)));
    pt_order_dev_ = pt_order + p0;  // this rank's internal points -> point ids
    k_col_free<<<grid_for(ncols_), 256, 0, s_>>>(static_cast<uint32_t>(nc), static_cast<uint32_t>(npl), cfix, pfix,
                                                 pt_order_dev_, col_free);
    CK(cudaGetLastError());
    classify_tiles(act_);
    d.normal_tiles = to_dev(b_normal_, act_.normal_tiles);
    d.heavy_tiles = to_dev(b_heavy_, act_.heavy_tiles);
    d.n_normal = static_cast<uint32_t>(act_.normal_tiles.size());
    d.n_heavy = static_cast<uint32_t>(act_.heavy_tiles.size());
    d.d_cam = d_cam;
    d.d_lpt = d_lpt;
    d.d_lcam = d_lcam;
    d.d_obs = d_obs;
    d.tile_cam_off = tile_cam_off;
    d.tile_cams = tile_cams;
    d.chunk_part_base = chunk_part_base;
    d.pt_slot_off = pt_slot_off;
    d.pt_slots = pt_slots;
    d.cam_part_off = cam_part_off;
    d.cam_part_idx = cam_part_idx;
    d.col_free = col_free;
    CK(cudaStreamSynchronize(s_));  // scratch buffers are released on return
    ptm.mark("act: runs, slots, csr");
  }

  void allocate_work() {
    const uint64_t nc = act_.nc, np = act_.np, ns = act_.n_slots;
    Dev<FP, SP>& d = dev_;
    int optin = 0;
    CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, g_.device));
    // recompute HVP (hvp_rc.cuh): analytic with SP == FP, or dynamic
    // in any precision, with the full-system PCG; no Jacobian store at all.
    // GB_HVP_RC=0 keeps the stored J (dynamic: the per-tile recompute kernel).
    rc_ok_ = false;
    if (g_.diff_mode != GB_AUTO && (std::is_same<SP, FP>::value || g_.diff_mode == GB_DYNAMIC) &&
        g_.linear_solver != GB_SOLVER_SCHUR && d.n_normal > 0) {
      rc_ = rc_layout<FP>(g_.loss_kind == GB_LOSS_HUBER, static_cast<uint32_t>(optin));
      rc_ok_ = rc_.ring_bytes >= rc_.max_region;  // any single tile fits (the ring drains before a huge one)
      if (const char* e = std::getenv("GB_HVP_RC")) rc_ok_ = rc_ok_ && std::atoi(e) != 0;
      if (const char* e = std::getenv("GB_RC_DBG")) rc_.dbg = std::atoi(e);
      // x += alpha p deferred into the next HVP (the fused direction update path only)
      d.defer_x = rc_ok_ && !fused_pcg_ ? 1 : 0;
      if (const char* e = std::getenv("GB_DEFER_X")) d.defer_x = d.defer_x && std::atoi(e) != 0;
      rc_.prof = nullptr;
      if (rc_.dbg & 8) {
        rc_.prof = static_cast<unsigned long long*>(b_rcprof_.alloc(16 * sizeof(unsigned long long)));
        CK(cudaMemsetAsync(rc_.prof, 0, 16 * sizeof(unsigned long long), s_));
      }
    }
    const bool dyn = g_.diff_mode == GB_DYNAMIC || rc_ok_;
    // factored J store: analytic mode with SP == FP; GB_JFACT=0 disables
    d.jfact = (!dyn && g_.diff_mode == GB_ANALYTIC && std::is_same<SP, FP>::value) ? 1 : 0;
    if (const char* e = std::getenv("GB_JFACT")) d.jfact = d.jfact && std::atoi(e) != 0;
    const uint64_t jrows = d.jfact ? kJFactRows : 24;
    const uint64_t jbytes = jstore_elems<SP>(ns, static_cast<int>(jrows)) * sizeof(SP);
    d.J = dyn ? nullptr : static_cast<SP*>(b_J_.alloc(jbytes));
    if (d.J) CK(cudaMemsetAsync(d.J, 0, jbytes, s_));  // padding slots stay 0
    d.Rf = d.jfact ? static_cast<FP*>(b_Rf_.alloc(std::max<uint64_t>(1, 10 * nc) * sizeof(FP))) : nullptr;
    d.cpre = static_cast<FP*>(b_cpre_.alloc(std::max<uint64_t>(1, kCamPre * nc) * sizeof(FP)));
    d.cpre_new = static_cast<FP*>(b_cpre_new_.alloc(std::max<uint64_t>(1, kCamPre * nc) * sizeof(FP)));
    d.w = g_.loss_kind == GB_LOSS_HUBER ? static_cast<FP*>(b_w_.alloc(ns * sizeof(FP))) : nullptr;
    if (d.w) CK(cudaMemsetAsync(d.w, 0, ns * sizeof(FP), s_));
    d.loss_kind = g_.loss_kind;
    d.huber = static_cast<FP>(g_.huber);
    // bulk-copy pipelined HVP (hvp_pipe.cuh): stored J, >= 2 stages in shared memory; GB_HVP_PIPE=0 disables
    {
      pipe_ = pipe_layout<FP, SP>(d.jfact ? kJFactRows : 24, d.w != nullptr, d.jfact != 0,
                                  static_cast<uint32_t>(optin));
      pipe_ok_ = d.J != nullptr && pipe_.stages >= 2 && d.n_normal > 0;
      if (const char* e = std::getenv("GB_HVP_PIPE")) pipe_ok_ = pipe_ok_ && std::atoi(e) != 0;
      if (const char* e = std::getenv("GB_PIPE_DBG")) pipe_.dbg = std::atoi(e);
      d.tile_meta = nullptr;
      d.tcv = nullptr;
      d.tile_aux = nullptr;
      d.slot_span = nullptr;
      d.tile_lin = nullptr;
      d.ntcams = act_.tile_cam_off.empty() ? 0 : act_.tile_cam_off.back();
      d.crec = d.part15 = nullptr;
      d.hflag = nullptr;
      d.lpart = nullptr;
      if (pipe_ok_ || rc_ok_) {
        if (pipe_ok_)
          CK(cudaFuncSetAttribute(k_hvp_pipe<FP, SP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(pipe_.total_bytes)));
        else if constexpr (kRcCapable)
          for (auto fn : {k_hvp_rc<FP, SP, false>, k_hvp_rc<FP, SP, true>})
            CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(rc_.total_bytes)));
        // tile records with the aux / lin blob offsets (16-byte units)
        std::vector<uint32_t> meta(static_cast<size_t>(kMCount) * d.n_normal, 0);
        uint64_t aux16 = 0, lin16 = 0;
        for (uint32_t i = 0; i < d.n_normal; ++i) {
          const uint32_t t = act_.normal_tiles[i];
          uint32_t* m = &meta[static_cast<size_t>(kMCount) * i];
          const uint32_t ne = act_.tile_ecnt[t], npt = act_.tile_pbeg[t + 1] - act_.tile_pbeg[t];
          const uint32_t ncam = act_.tile_cam_off[t + 1] - act_.tile_cam_off[t];
          m[kMT] = t;
          m[kMEb] = act_.tile_ebeg[t];
          m[kMNe] = ne;
          m[kMPb] = act_.tile_pbeg[t];
          m[kMNpt] = npt;
          m[kMCb] = act_.tile_cam_off[t];
          m[kMNcam] = ncam;
          m[kMCh0] = act_.tile_chunk_base[t];
          if (rc_ok_) {  // one blob per tile: static aux part, then the per-linearization part (one bulk copy)
            m[kMAux16] = static_cast<uint32_t>(aux16);
            aux16 += aux_sections(ne, npt).bytes / 16;
            m[kMLin16] = static_cast<uint32_t>(aux16);
            aux16 += rc_lin_sections<FP>(ne, npt, ncam, d.w != nullptr).bytes / 16;
          } else {
            m[kMAux16] = static_cast<uint32_t>(aux16);
            m[kMLin16] = static_cast<uint32_t>(lin16);
            aux16 += aux_sections(ne, npt).bytes / 16;
            lin16 += lin_sections<FP>(ne, npt, ncam, d.jfact != 0, d.w != nullptr).bytes / 16;
          }
        }
        if (aux16 > 0xffffffffull || lin16 > 0xffffffffull) throw std::invalid_argument("tile blobs exceed 64 GB");
        d.tile_meta = to_dev(b_tmeta_, meta);
        d.tile_aux = static_cast<unsigned char*>(b_taux_.alloc(std::max<uint64_t>(16, 16 * aux16)));
        d.slot_span = static_cast<uint2*>(b_sspan_.alloc(std::max<uint64_t>(8, 8ull * act_.nparts)));
        d.tile_lin = rc_ok_ ? d.tile_aux : static_cast<unsigned char*>(b_tlin_.alloc(std::max<uint64_t>(16, 16 * lin16)));
        if (pipe_ok_) {
          d.tcv = static_cast<A*>(b_tcv_.alloc(std::max<uint64_t>(1, cam_stride<A>() * uint64_t(d.ntcams)) * sizeof(A)));
          CK(cudaMemsetAsync(d.tcv, 0, std::max<uint64_t>(1, cam_stride<A>() * uint64_t(d.ntcams)) * sizeof(A), s_));
        } else {
          const uint64_t nt = std::max<uint64_t>(1, d.ntcams);
          d.crec = static_cast<FP*>(b_crec_.alloc(std::max<uint64_t>(1, nc) * kRcRec * sizeof(FP)));
          d.part15 = static_cast<FP*>(b_part15_.alloc(nt * kRcRec * sizeof(FP)));
          CK(cudaMemsetAsync(d.part15, 0, nt * kRcRec * sizeof(FP), s_));  // heavy tiles' entries stay 0
          uint8_t* hf = static_cast<uint8_t*>(b_hflag_.alloc(std::max<uint64_t>(1, act_.nparts)));
          CK(cudaMemsetAsync(hf, 0, std::max<uint64_t>(1, act_.nparts), s_));
          d.hflag = hf;
          // linearize camera-run sums per tile camera (k_lin_seg); heavy tiles' entries stay 0
          bool seg = g_.diff_mode != GB_AUTO;
          if (const char* e = std::getenv("GB_LIN_SEG")) seg = seg && std::atoi(e) != 0;
          if (seg) {
            d.lpart = static_cast<FP*>(b_lpart_.alloc(nt * kLinVals * sizeof(FP)));
            CK(cudaMemsetAsync(d.lpart, 0, nt * kLinVals * sizeof(FP), s_));
            CK(cudaFuncSetAttribute(k_lin_seg<FP, SP, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(lin_seg_smem<FP>())));
            CK(cudaFuncSetAttribute(k_lin_seg<FP, SP, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(lin_seg_smem<FP>())));
          }
        }
        pipe_aux_pending_ = true;  // built once the remaining device arrays exist (below)
      }
    }
    d.part = static_cast<FP*>(b_part_.alloc(std::max<uint64_t>(1, act_.nparts) * kLinVals * sizeof(FP)));
    {  // camera-major storage of the partial slots: run -> its position in the camera lists
      uint32_t* rs = static_cast<uint32_t*>(b_runslot_.alloc(std::max<uint64_t>(1, act_.nparts) * sizeof(uint32_t)));
      if (act_.nparts) k_run_slots<<<grid_for(act_.nparts), 256, 0, s_>>>(act_.nparts, d.cam_part_idx, rs);
      CK(cudaGetLastError());
      d.run_slot = rs;
    }
    d.x = static_cast<FP*>(b_x_.alloc(ncols_ * sizeof(FP)));
    d.x_new = static_cast<FP*>(b_xn_.alloc(ncols_ * sizeof(FP)));
    d.b = static_cast<FP*>(b_b_.alloc(ncols_ * sizeof(FP)));
    d.clamped = static_cast<FP*>(b_cl_.alloc(ncols_ * sizeof(FP)));
    d.D = static_cast<FP*>(b_D_.alloc(ncols_ * sizeof(FP)));
    d.dx = static_cast<FP*>(b_dx_.alloc(ncols_ * sizeof(FP)));
    d.Hc = static_cast<FP*>(b_Hc_.alloc(45 * nc * sizeof(FP)));
    d.Hp = static_cast<FP*>(b_Hp_.alloc(6 * np * sizeof(FP)));
    d.Mc = static_cast<FP*>(b_Mc_.alloc(45 * nc * sizeof(FP)));
    d.Mp = static_cast<FP*>(b_Mp_.alloc(6 * np * sizeof(FP)));
    d.xs = static_cast<SP*>(b_xs_.alloc(ncols_ * sizeof(SP)));
    d.r = static_cast<SP*>(b_r_.alloc(ncols_ * sizeof(SP)));
    d.z = static_cast<SP*>(b_z_.alloc(ncols_ * sizeof(SP)));
    d.p = static_cast<SP*>(b_p_.alloc(ncols_ * sizeof(SP)));
    d.ap = static_cast<SP*>(b_ap_.alloc(ncols_ * sizeof(SP)));
    d.vt = static_cast<A*>(b_vt_.alloc(ncols_ * sizeof(A)));
    CK(cudaMemsetAsync(d.vt, 0, ncols_ * sizeof(A), s_));
    d.rc = static_cast<FP*>(b_rc_.alloc(std::max<uint64_t>(1, 9 * nc) * sizeof(FP)));
    d.xp = static_cast<FP*>(b_xp_.alloc(std::max<uint64_t>(1, 3 * np) * sizeof(FP)));
    d.tile_red = static_cast<FP*>(b_tr_.alloc(8ull * act_.ntiles * sizeof(FP)));
    d.tile_red2 = static_cast<FP*>(b_tr2_.alloc(act_.ntiles * sizeof(FP)));
    d.tile_flag = static_cast<int*>(b_tf_.alloc(act_.ntiles * sizeof(int)));
    d.cam_red = static_cast<FP*>(b_cr_.alloc(std::max<uint64_t>(1, nc) * sizeof(FP)));
    const uint64_t nblk =
        std::max<uint64_t>(std::max<uint64_t>(std::max<uint64_t>(std::max<uint64_t>(vert_grid(), col_grid()), cam_grid()),
                                              coop_grid_),
                           chi2_grid()) +
        pt_grid();
    d.blk_red = static_cast<FP*>(b_br_.alloc(nblk * sizeof(FP)));
    d.blk_red2 = static_cast<FP*>(b_br2_.alloc(nblk * sizeof(FP)));
    d.blk_flag = static_cast<int*>(b_bf_.alloc(nblk * sizeof(int)));
    d.st = st_;
    d.recs = rec_buf_.as<gb_iteration_record>();
    d.world = g_.world();
    d.rank = g_.rank();
    d.dist = g_.reducer ? 1 : 0;
    d.red = static_cast<FP*>(b_red_.alloc((54ull * nc + 8 + kRedCount + 8) * sizeof(FP)));
    d.redmax = static_cast<FP*>(b_redmax_.alloc(8 * sizeof(FP)));
    CK(cudaMemsetAsync(d.red, 0, (54ull * nc + 8 + kRedCount + 8) * sizeof(FP), s_));
    CK(cudaMemsetAsync(d.redmax, 0, 8 * sizeof(FP), s_));
    CK(cudaMemsetAsync(d.xs, 0, ncols_ * sizeof(SP), s_));
    CK(cudaMemsetAsync(d.p, 0, ncols_ * sizeof(SP), s_));
    b_ptstage_.alloc(std::max<uint64_t>(1, 3 * np) * sizeof(FP));
    if (pipe_aux_pending_) {
      // camera -> tile-camera entries (stable by entry index) for k_pcg_dir_rest's tcv scatter
      {
        using namespace actdev;
        const uint64_t nt = d.ntcams;
        DBuf s_keys, s_vals, s_keys2, s_cnt;
        uint32_t* vals = scratch<uint32_t>(s_vals, nt);
        uint32_t* keys2 = scratch<uint32_t>(s_keys2, nt);
        uint32_t* idx = static_cast<uint32_t*>(b_camtc_idx_.alloc(std::max<uint64_t>(1, nt) * sizeof(uint32_t)));
        k_iota<<<grid_for(nt), 256, 0, s_>>>(nt, vals);
        cub_sort<uint32_t>(d.tile_cams, keys2, vals, idx, nt, bits_for(nc));
        uint32_t* cnt = scratch<uint32_t>(s_cnt, nc + 1);
        CK(cudaMemsetAsync(cnt, 0, (nc + 1) * sizeof(uint32_t), s_));
        k_hist<<<grid_for(nt), 256, 0, s_>>>(nt, d.tile_cams, cnt);
        uint32_t* off = static_cast<uint32_t*>(b_camtc_off_.alloc((nc + 1) * sizeof(uint32_t)));
        cub_scan_excl(cnt, off, nc + 1);
        d.cam_tc_off = off;
        d.cam_tc_idx = idx;
        CK(cudaStreamSynchronize(s_));
      }
      // point columns of heavy tiles (k_pcg_dir_rest applies p = z + beta p there)
      {
        std::vector<uint64_t> rb, re;
        for (uint32_t t : act_.heavy_tiles) {
          const uint64_t c0 = 9ull * nc + 3ull * act_.tile_pbeg[t], c1 = 9ull * nc + 3ull * act_.tile_pbeg[t + 1];
          if (!re.empty() && re.back() == c0)
            re.back() = c1;
          else {
            rb.push_back(c0);
            re.push_back(c1);
          }
        }
        dir_nranges_ = static_cast<int>(rb.size());
        dir_rbeg_ = to_dev(b_dir_rb_, rb);
        dir_rend_ = to_dev(b_dir_re_, re);
        uint64_t work = 9ull * nc;
        for (size_t r = 0; r < rb.size(); ++r) work += re[r] - rb[r];
        dir_rest_grid_ = grid_for(work);
      }
      k_tile_aux<FP, SP><<<d.n_normal, 256, 0, s_>>>(d);
      CK(cudaGetLastError());
      if (rc_ok_ && d.n_heavy) {
        k_mark_heavy_slots<FP, SP><<<d.n_heavy, 256, 0, s_>>>(d, const_cast<uint8_t*>(d.hflag));
        CK(cudaGetLastError());
      }
      pipe_aux_pending_ = false;
    }
  }

  // user AoS -> internal order on the device (cameras copied as is)
  void upload_params() {
    const uint64_t nc = act_.nc, np = act_.np;
    FP* stage = b_ptstage_.as<FP>();
    CK(cudaMemcpyAsync(dev_.x, g_.cams, 9 * nc * sizeof(FP), cudaMemcpyHostToDevice, s_));
    // every user point is staged (a shard gathers its own internal range:
    // pt_order_dev_ points at it)
    const uint64_t np_all = g_.np;
    if (!pts_staged_) {  // else already uploaded under the device activation (s_ waited on ev_up_)
      stage = static_cast<FP*>(b_ptstage_.alloc(std::max<uint64_t>(1, 3 * np_all) * sizeof(FP)));
      if (np_all) CK(cudaMemcpyAsync(stage, g_.pts, 3 * np_all * sizeof(FP), cudaMemcpyHostToDevice, s_));
    }
    actdev::k_gather_points<FP><<<grid_for(3 * np), 256, 0, s_>>>(static_cast<uint32_t>(np), pt_order_dev_, stage,
                                                                  dev_.x + 9 * nc);
    CK(cudaGetLastError());
    pts_staged_ = false;
    h2d_bytes_ += (9 * nc + 3 * np_all) * sizeof(FP);
  }

  void download_params() {
    if (dist()) {
      download_params_sharded();
      return;
    }
    const uint64_t nc = act_.nc, np = act_.np;
    FP* stage = b_ptstage_.as<FP>();
    actdev::k_scatter_points<FP><<<grid_for(3 * np), 256, 0, s_>>>(static_cast<uint32_t>(np), pt_order_dev_,
                                                                   dev_.x + 9 * nc, stage);
    CK(cudaGetLastError());
    // fixed vertices are written back with their own bits (bit-identical)
    CK(cudaMemcpyAsync(g_.cams, dev_.x, 9 * nc * sizeof(FP), cudaMemcpyDeviceToHost, s_));
    CK(cudaMemcpyAsync(g_.pts, stage, 3 * np * sizeof(FP), cudaMemcpyDeviceToHost, s_));
    CK(cudaStreamSynchronize(s_));
    d2h_bytes_ += ncols_ * sizeof(FP);
  }

  // every rank ends with every point: each shard broadcasts its internal point
  // range (bit-exact copies, fixed points included)
  void download_params_sharded() {
    const uint64_t nc = act_.nc;
    FP* xall = static_cast<FP*>(b_xall_.alloc(std::max<uint64_t>(1, 3 * full_np_) * sizeof(FP)));
    const int me = g_.rank();
    CK(cudaMemcpyAsync(xall + 3ull * shard_p0_[me], dev_.x + 9 * nc, 3ull * act_.np * sizeof(FP),
                       cudaMemcpyDeviceToDevice, s_));
    for (int r = 0; r < g_.world(); ++r) {
      const uint64_t n = 3ull * (shard_p0_[r + 1] - shard_p0_[r]);
      if (n) g_.reducer->broadcast(xall + 3ull * shard_p0_[r], n * sizeof(FP), r, s_);
    }
    std::vector<FP> hc(9 * nc), hp(3 * full_np_);
    CK(cudaMemcpyAsync(hc.data(), dev_.x, hc.size() * sizeof(FP), cudaMemcpyDeviceToHost, s_));
    CK(cudaMemcpyAsync(hp.data(), xall, hp.size() * sizeof(FP), cudaMemcpyDeviceToHost, s_));
    CK(cudaStreamSynchronize(s_));
    d2h_bytes_ += (hc.size() + hp.size()) * sizeof(FP);
    std::memcpy(g_.cams, hc.data(), hc.size() * sizeof(FP));
    FP* up = static_cast<FP*>(g_.pts);
    for (uint64_t i = 0; i < full_np_; ++i) {
      const uint64_t p = full_pt_order_[i];
      up[3 * p] = hp[3 * i];
      up[3 * p + 1] = hp[3 * i + 1];
      up[3 * p + 2] = hp[3 * i + 2];
    }
  }

  void fill_config(State<FP>& hs, const gb_lm_config& cfg) {
    hs.tol = cfg.tolerance;
    hs.grad_tol = cfg.gradient_tolerance;
    hs.lambda_max = cfg.lambda_max;
    hs.tau = cfg.tau;
    hs.pcg_tol = cfg.pcg.tolerance;
    hs.pcg_ratio = cfg.pcg.rejection_ratio;
    hs.pcg_max_it = cfg.pcg.max_iterations;
    hs.normalize_rhs = cfg.pcg.normalize_rhs;
    hs.clamp_min = cfg.clamp_min;
    hs.clamp_max = cfg.clamp_max;
    hs.before_scaling = cfg.damping == GB_DAMPING_BEFORE_SCALING;
    hs.use_guard = cfg.use_rejection_guard;
    hs.refresh_on_reject = cfg.refresh_on_reject;
    hs.max_iterations = cfg.max_iterations;
    hs.schur = g_.linear_solver == GB_SOLVER_SCHUR ? 1 : 0;
    if (hs.schur && g_.diff_mode == GB_DYNAMIC)
      throw std::invalid_argument("Schur mode needs stored Jacobians (analytic or auto)");
    if (hs.schur && g_.reducer) throw std::logic_error("Schur mode is single-GPU in this build");
  }

  // ------------------------------------------------------------- launches
  // one vertex per thread (memory-level parallelism beats grid-stride reuse here)

  // one full wave of the point kernels (occupancy measured once per solver)
  unsigned chi2_grid() const { return std::max(1u, std::min(act_.ntiles, sms_ * chi2_occ_)); }
  unsigned pt_grid() const { return std::max(1u, std::min(div_up(act_.np, 256), sms_ * pt_occ_)); }
  void launch_pcg_init() {
    k_pcg_init<FP, SP><<<vert_grid(), 256, 0, s_>>>(dev_);
    CK(cudaGetLastError());
  }
  void launch_pcg_update() {
    // 8-byte storage: a resident grid of 4 CTAs per SM (64-register bound); else the vertex grid
    const unsigned g = sizeof(SP) == 8 ? std::min(vert_grid(), sms_ * 4u) : vert_grid();
    k_pcg_update<FP, SP><<<g, 256, 0, s_>>>(dev_);
    CK(cudaGetLastError());
  }
  void launch_precond() {
    k_precond_cams<FP, SP><<<std::max(1u, div_up(act_.nc, 64)), 64, 0, s_>>>(dev_);
    k_precond_pts<FP, SP><<<pt_grid(), 256, 0, s_>>>(dev_);
    CK(cudaGetLastError());
  }
  unsigned vert_grid() const {
    return std::max(1u, std::min(div_up(static_cast<uint64_t>(act_.nc) + act_.np, 256), sms_ * 6u));
  }
  unsigned col_grid() const { return std::max(1u, std::min(div_up(ncols_, 256), 148u * 8u)); }
  unsigned cam_grid() const { return std::max(1u, div_up(act_.nc, kCamWarps)); }

  // ---- collectives (world > 1)
  bool dist() const { return static_cast<bool>(g_.reducer); }
  void allreduce(FP* p, size_t n, bool max = false) {
    g_.reducer->allreduce(p, n, static_cast<int>(sizeof(FP)), max, s_);
  }
  FP* red_s() const { return dev_.red + red_scalars(dev_); }
  void fin(int site) {
    k_fin<FP, SP><<<1, 1, 0, s_>>>(dev_, site);
    CK(cudaGetLastError());
  }

  void enqueue_linearize(int force) {
    const size_t smem = lin_normal_smem<FP>();
    k_cam_pre<FP, SP><<<std::max(1u, div_up(act_.nc, 128)), 128, 0, s_>>>(dev_, dev_.x, dev_.cpre, 0, force);
    const bool aut = g_.diff_mode == GB_AUTO;
    phase_mark("lin: k_cam_pre");
    if (dev_.J && aut) {  // Auto: stored J from dual-number passes (factor_descriptor.hpp:610-624)
      if (dev_.n_normal) k_lin_normal<FP, SP, true, true><<<dev_.n_normal, kLinThreads, smem, s_>>>(dev_, force);
      if (dev_.n_heavy)
        k_lin_tiles<FP, SP, true, true><<<dev_.n_heavy, kTileThreads, 0, s_>>>(dev_, dev_.heavy_tiles, force);
    } else if (dev_.J) {
      if (dev_.n_normal) k_lin_normal<FP, SP, true, false><<<dev_.n_normal, kLinThreads, smem, s_>>>(dev_, force);
      if (dev_.n_heavy)
        k_lin_tiles<FP, SP, true, false><<<dev_.n_heavy, kTileThreads, 0, s_>>>(dev_, dev_.heavy_tiles, force);
    } else {
      if (dev_.n_normal && dev_.lpart)
        if (dev_.w)
          k_lin_seg<FP, SP, true><<<dev_.n_normal, kLinSegThreads, lin_seg_smem<FP>(), s_>>>(dev_, force);
        else
          k_lin_seg<FP, SP, false><<<dev_.n_normal, kLinSegThreads, lin_seg_smem<FP>(), s_>>>(dev_, force);
      else if (dev_.n_normal)
        k_lin_normal<FP, SP, false, false><<<dev_.n_normal, kLinThreads, smem, s_>>>(dev_, force);
      if (dev_.n_heavy)
        k_lin_tiles<FP, SP, false, false><<<dev_.n_heavy, kTileThreads, 0, s_>>>(dev_, dev_.heavy_tiles, force);
    }
    CK(cudaGetLastError());
    phase_mark("lin: tiles");
    if (!dist()) {
      k_lin_cams<FP, SP><<<cam_grid(), 32 * kCamWarps, 0, s_>>>(dev_, force, 0);
    } else {
      k_lin_cams<FP, SP><<<cam_grid(), 32 * kCamWarps, 0, s_>>>(dev_, force, 1);
      CK(cudaGetLastError());
      allreduce(dev_.red, red_scalars(dev_) + 2);
      allreduce(dev_.redmax + kRedMaxLin, 1, true);
      k_lin_cams<FP, SP><<<cam_grid(), 32 * kCamWarps, 0, s_>>>(dev_, force, 2);
    }
    CK(cudaGetLastError());
    if (pipe_ok_) {
      k_tile_lin<FP, SP><<<dev_.n_normal, 128, 0, s_>>>(dev_, force);
      CK(cudaGetLastError());
    } else if (rc_ok_ && (g_.diff_mode == GB_AUTO || !dev_.part15)) {  // else k_lin_normal wrote the blobs
      phase_mark("lin: cameras");
      k_tile_lin_rc<FP, SP><<<dev_.n_normal, 128, 0, s_>>>(dev_, force);
      CK(cudaGetLastError());
    }
  }

  // HVP tile pass (dynamic mode recomputes J per edge).
  // tcv_ready: the stored-J pipeline's per-tile camera copies are current
  // (k_pcg_dir_rest ran); on the recompute path it means the direction update
  // p = z + beta p is pending and is applied here (cameras, heavy-tile points)
  // and inside k_hvp_rc (normal-tile points).
  void launch_hvp_tiles(const Dev<FP, SP>& d, bool tcv_ready = false) {
    if constexpr (kRcCapable) {
      if (rc_ok_) {
        launch_hvp_rc(d, tcv_ready);
        return;
      }
    }
    if (!d.J) {
      k_hvp_tiles<FP, SP, true><<<act_.ntiles, kTileThreads, 0, s_>>>(d, nullptr);
    } else if (pipe_ok_) {  // normal tiles through the bulk-copy pipeline, heavy tiles one CTA each
      if (!tcv_ready) k_tcam_vt<FP, SP><<<grid_for(cam_stride<A>() * uint64_t(d.ntcams)), 256, 0, s_>>>(d);
      k_hvp_pipe<FP, SP><<<std::min<uint32_t>(d.n_normal, sms_), kPipeThreads, pipe_.total_bytes, s_>>>(d, pipe_);
      if (d.n_heavy) k_hvp_tiles<FP, SP, false, 1><<<d.n_heavy, kTileThreads, 0, s_>>>(d, d.heavy_tiles);
    } else if (hvp_minb_ == 4) {
      k_hvp_tiles<FP, SP, false, 4><<<act_.ntiles, kTileThreads, 0, s_>>>(d, nullptr);
    } else {
      k_hvp_tiles<FP, SP, false, 1><<<act_.ntiles, kTileThreads, 0, s_>>>(d, nullptr);
    }
    CK(cudaGetLastError());
  }

  // recompute HVP (hvp_rc.cuh): camera records (+ direction update), the tile
  // pipeline (which gathers them per tile), heavy tiles with the dynamic tile kernel
  void launch_hvp_rc(const Dev<FP, SP>& d, bool dir) {
    k_rc_cams_pre<FP, SP><<<std::max(1u, div_up(act_.nc, 128)), 128, 0, s_>>>(d, dir ? 1 : 0, dir_rbeg_, dir_rend_,
                                                                              dir_nranges_);
    const uint32_t grid = std::min<uint32_t>(d.n_normal, sms_);
    if (d.w)
      k_hvp_rc<FP, SP, true><<<grid, kRcThreadsWS, rc_.total_bytes, s_>>>(d, rc_);
    else
      k_hvp_rc<FP, SP, false><<<grid, kRcThreadsWS, rc_.total_bytes, s_>>>(d, rc_);
    if (d.n_heavy) k_hvp_tiles<FP, SP, true, 1><<<d.n_heavy, kTileThreads, 0, s_>>>(d, d.heavy_tiles);
    CK(cudaGetLastError());
  }

  void launch_hvp(const Dev<FP, SP>& d, bool tcv_ready = false) {
    launch_hvp_tiles(d, tcv_ready);
    if (rc_ok_) {
      if constexpr (kRcCapable) {
        if (!dist()) {
          k_hvp_cams_rc<FP, SP><<<std::max(1u, div_up(act_.nc, kRcCamsPerBlock)), 16 * kRcCamsPerBlock, 0, s_>>>(d, 0);
        } else {
          k_hvp_cams_rc<FP, SP><<<std::max(1u, div_up(act_.nc, kRcCamsPerBlock)), 16 * kRcCamsPerBlock, 0, s_>>>(d, 1);
          CK(cudaGetLastError());
          allreduce(d.red, 9ull * d.nc + 1);
          k_hvp_cams_rc<FP, SP><<<std::max(1u, div_up(act_.nc, kRcCamsPerBlock)), 16 * kRcCamsPerBlock, 0, s_>>>(d, 2);
        }
      }
    } else if (!dist()) {
      k_hvp_cams<FP, SP><<<cam_grid(), 32 * kCamWarps, 0, s_>>>(d, 0);
    } else {
      k_hvp_cams<FP, SP><<<cam_grid(), 32 * kCamWarps, 0, s_>>>(d, 1);
      CK(cudaGetLastError());
      allreduce(d.red, 9ull * d.nc + 1);
      k_hvp_cams<FP, SP><<<cam_grid(), 32 * kCamWarps, 0, s_>>>(d, 2);
    }
    CK(cudaGetLastError());
  }

  // Schur mode (kernels.cuh k_schur_*): camera blocks of S, reduced rhs, PCG
  // on the cameras, back-substitution of the points, step.
  void enqueue_solve_schur(int pcg_max_it) {
    launch_precond();  // point blocks = A_pp^-1
    k_schur_pre_tiles<FP, SP><<<act_.ntiles, kTileThreads, 0, s_>>>(dev_);
    k_schur_pre_cams<FP, SP><<<div_up(act_.nc, 128), 128, 0, s_>>>(dev_);
    k_schur_tiles<FP, SP, 1><<<act_.ntiles, kTileThreads, 0, s_>>>(dev_);
    k_schur_rhs_cams<FP, SP><<<cam_grid(), 32 * kCamWarps, 0, s_>>>(dev_);
    k_rhs_norm<FP, SP><<<col_grid(), 256, 0, s_>>>(dev_);
    launch_pcg_init();
    CK(cudaGetLastError());
    for (int k = 0; k < pcg_max_it; ++k) {
      k_schur_tiles<FP, SP, 0><<<act_.ntiles, kTileThreads, 0, s_>>>(dev_);
      k_hvp_cams<FP, SP><<<cam_grid(), 32 * kCamWarps, 0, s_>>>(dev_, 0);
      if (fused_pcg_) {
        launch_pcg_step();
      } else {
        launch_pcg_update();
        k_pcg_dir<FP, SP><<<col_grid(), 256, 0, s_>>>(dev_);
      }
      CK(cudaGetLastError());
    }
    k_schur_xc<FP, SP><<<col_grid(), 256, 0, s_>>>(dev_);
    k_schur_tiles<FP, SP, 2><<<act_.ntiles, kTileThreads, 0, s_>>>(dev_);
    k_step<FP, SP><<<col_grid(), 256, 0, s_>>>(dev_);
    CK(cudaGetLastError());
  }

  void launch_pcg_step() {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(coop_grid_);
    cfg.blockDim = dim3(256);
    cfg.stream = s_;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, k_pcg_step<FP, SP>, dev_));
  }

  // build_preconditioner + pcg_solve + unscale (linear_system.hpp:185-207)
  void enqueue_solve(int pcg_max_it) {
    if (g_.linear_solver == GB_SOLVER_SCHUR) {
      enqueue_solve_schur(pcg_max_it);
      return;
    }
    launch_precond();
    CK(cudaGetLastError());
    phase_mark("solve: precond");
    k_rhs_norm<FP, SP><<<col_grid(), 256, 0, s_>>>(dev_);
    CK(cudaGetLastError());
    if (dist()) {
      allreduce(red_s() + kRedRhs, 2);
      fin(1);
    }
    launch_pcg_init();
    CK(cudaGetLastError());
    if (dist()) {
      allreduce(red_s() + kRedInitRz, 2);
      fin(2);
    }
    const bool dir_fused = (pipe_ok_ || rc_ok_) && !(!dist() && fused_pcg_);
    phase_mark("solve: rhs + init");
    for (int k = 0; k < pcg_max_it; ++k) {
      launch_hvp(dev_, dir_fused && k > 0);  // after k_pcg_dir_rest the per-tile camera copies are current
      phase_mark("solve: HVP");
      if (!dist() && fused_pcg_) {
        launch_pcg_step();
        continue;
      }
      launch_pcg_update();
      CK(cudaGetLastError());
      if (dist()) {
        allreduce(red_s() + kRedUpdRz, 2);
        fin(3);
      }
      if (rc_ok_ && dir_fused)  // applied by the next launch_hvp (k_rc_cams_pre + k_hvp_rc)
        ;
      else if (dir_fused)  // normal-tile points get p = z + beta p inside the next k_hvp_pipe
        k_pcg_dir_rest<FP, SP><<<dir_rest_grid_, 256, 0, s_>>>(dev_, dir_rbeg_, dir_rend_, dir_nranges_);
      else
        k_pcg_dir<FP, SP><<<col_grid(), 256, 0, s_>>>(dev_);
      CK(cudaGetLastError());
      phase_mark("solve: update");
    }
    k_step<FP, SP><<<col_grid(), 256, 0, s_>>>(dev_);
    CK(cudaGetLastError());
    if (dist()) {
      allreduce(red_s() + kRedStepPred, 2);
      fin(4);
    }
  }

  // One LM iteration (levenberg_marquardt.hpp:149-220) as a fixed kernel
  // sequence; every kernel early-exits on the device flags it depends on.
  void enqueue_iteration(int pcg_max_it) {
    phase_mark(nullptr);
    k_iter_begin<FP><<<1, 1, 0, s_>>>(st_, dev_.recs);
    CK(cudaGetLastError());
    enqueue_solve(pcg_max_it);
    phase_mark("solve: step");
    k_cam_pre<FP, SP><<<std::max(1u, div_up(act_.nc, 128)), 128, 0, s_>>>(dev_, dev_.x_new, dev_.cpre_new, 1, 0);
    k_chi2_tiles<FP, SP, false><<<chi2_grid(), kTileThreads, 0, s_>>>(dev_, dev_.x_new, 0);
    CK(cudaGetLastError());
    if (dist()) {
      allreduce(red_s() + kRedChi, 1);
      fin(5);
    }
    phase_mark("candidate chi2");
    k_decide<FP><<<1, 1, 0, s_>>>(st_, dev_.recs);
    CK(cudaGetLastError());
    k_commit<FP, SP><<<col_grid(), 256, 0, s_>>>(dev_);
    CK(cudaGetLastError());
    phase_mark("decide + commit");
    enqueue_linearize(0);
    phase_mark("lin: tile blobs");
  }

  // GB_PHASES=1 (experiments): iterations run uncaptured with CUDA events
  // between phases; the mean device time per phase occurrence is printed when
  // the handle is destroyed
  void phase_mark(const char* name) {
    if (!phases_on_) return;
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    CK(cudaEventRecord(e, s_));
    phase_ev_.push_back({e, name});
  }
  void phase_flush() {
    if (phase_ev_.empty()) return;
    CK(cudaStreamSynchronize(s_));
    for (size_t i = 1; i < phase_ev_.size(); ++i) {
      if (!phase_ev_[i].second) continue;
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, phase_ev_[i - 1].first, phase_ev_[i].first));
      auto& acc = phase_ms_[phase_ev_[i].second];
      acc.first += ms;
      acc.second += 1;
    }
    for (auto& pe : phase_ev_) cudaEventDestroy(pe.first);
    phase_ev_.clear();
  }
  bool phases_on_ = std::getenv("GB_PHASES") != nullptr;
  std::vector<std::pair<cudaEvent_t, const char*>> phase_ev_;
  std::map<std::string, std::pair<double, int>> phase_ms_;

  void build_iteration_graph(int pcg_max_it) {
    if (graph_exec_ && graph_pcg_it_ == pcg_max_it && graph_recs_ == dev_.recs) return;
    if (graph_exec_) cudaGraphExecDestroy(graph_exec_);
    graph_exec_ = nullptr;
    cudaGraph_t graph;
    CK(cudaStreamBeginCapture(s_, cudaStreamCaptureModeThreadLocal));
    enqueue_iteration(pcg_max_it);
    CK(cudaStreamEndCapture(s_, &graph));
    // kernel nodes of one LM iteration (gb_iteration_kernels: bench.py's gpu_launches)
    size_t nn = 0;
    CK(cudaGraphGetNodes(graph, nullptr, &nn));
    std::vector<cudaGraphNode_t> nodes(nn);
    if (nn) CK(cudaGraphGetNodes(graph, nodes.data(), &nn));
    graph_kernels_ = 0;
    for (auto nd : nodes) {
      cudaGraphNodeType t;
      CK(cudaGraphNodeGetType(nd, &t));
      graph_kernels_ += t == cudaGraphNodeTypeKernel;
    }
    CK(cudaGraphInstantiate(&graph_exec_, graph, 0));
    CK(cudaGraphDestroy(graph));
    graph_pcg_it_ = pcg_max_it;
    graph_recs_ = dev_.recs;
  }

  gb_memory_account memory_account() const {
    // analytic account, levenberg_marquardt.hpp:100-108 and README "Memory accounting"
    struct LossFP {
      int kind;
      FP delta;
    };
    const uint64_t N = static_cast<uint64_t>(act_.free_dims);
    gb_memory_account m{};
    m.jacobian_bytes = g_.diff_mode == GB_DYNAMIC ? 0 : act_.n_active * 2 * 12 * sizeof(SP);
    m.preconditioner_bytes = (81ull * act_.free_cams + 9ull * act_.free_pts) * sizeof(FP);
    m.workspace_bytes = 5 * N * sizeof(SP) + 6 * N * sizeof(FP) + act_.n_active * (4 * sizeof(FP) + 2 * sizeof(A));
    const uint64_t vtx = sizeof(uint64_t) + sizeof(void*) + 1 + sizeof(int64_t);
    m.graph_bytes = g_.nc * (9 * sizeof(FP) + vtx) + g_.np * (3 * sizeof(FP) + vtx) +
                    g_.ne * (2 * sizeof(uint32_t) + 2 * sizeof(FP) + 1 + 4 * sizeof(FP) + sizeof(LossFP) + 1);
    return m;
  }

  GraphData& g_;
  cudaStream_t s_ = nullptr;
  cudaStream_t s_up_ = nullptr;  // side stream: the observation upload overlaps activation (device activation)
  cudaEvent_t ev_up_ = nullptr;
  bool pts_staged_ = false;      // the point parameters are already in b_ptstage_ (this begin's activation)
  // phase state of the current solve
  gb_lm_config cfg_{};
  gb_solve_report rep_{};
  bool in_solve_ = false;
  int max_it_ = 0, launched_ = 0, pcg_max_it_ = 0;
  std::vector<cudaEvent_t> ev_;
  Clock::time_point t0_;
  Activation act_;
  bool have_act_ = false;
  uint64_t act_rev_ = 0;
  int act_level_ = 0;
  uint64_t ncols_ = 0;
  std::vector<uint64_t> ref_to_int_;
  uint64_t full_np_ = 0;
  std::vector<uint32_t> full_pt_order_, shard_p0_;
  Dev<FP, SP> dev_{};
  State<FP>* st_ = nullptr;
  State<FP> ls_state_{};
  bool ls_ready_ = false;
  int* flag_host_ = nullptr;
  size_t h2d_bytes_ = 0, d2h_bytes_ = 0;
  cudaGraphExec_t graph_exec_ = nullptr;
  int graph_pcg_it_ = -1;
  int graph_kernels_ = 0;
  gb_iteration_record* graph_recs_ = nullptr;
  DBuf st_buf_, rec_buf_, dbg_buf_;
  DBuf b_rc_, b_xp_;
  DBuf b_red_, b_redmax_, b_xall_, b_pt_order_, b_da_, b_cub_, b_ptstage_;
  uint32_t* pt_order_dev_ = nullptr;
  bool host_plan_ = false;
  unsigned coop_grid_ = 148 * 8;  // co-resident blocks of k_pcg_step (cooperative launch)
  bool fused_pcg_ = false;  // GB_PCG_FUSED=1: cooperative k_pcg_step (measured slower: 358 vs 335 us at Final)
  int hvp_minb_ = 4;  // occupancy hint of the HVP tile kernel (A/B: GB_HVP_MINB=1 -> 80 regs, 3 CTAs/SM)
  DBuf b_vt_, b_dlcam_, b_tile_ecnt_, b_tile_cam_off_, b_tile_cams_, b_normal_, b_heavy_;
  DBuf b_col_free_, b_dcam_, b_dlpt_, b_obs_, b_tile_ebeg_, b_tile_pbeg_, b_tile_chunk_, b_chunk_part_,
      b_pt_slot_off_, b_pt_slots_, b_cam_part_off_, b_cam_part_idx_;
  PipeLayout pipe_{};
  bool pipe_ok_ = false;
  static constexpr bool kRcCapable = true;  // every precision (bf16 storage: dynamic mode only)
  RcLayout rc_{};
  bool rc_ok_ = false;  // recompute HVP (hvp_rc.cuh): no J store
  DBuf b_crec_, b_part15_, b_hflag_, b_rcprof_, b_lpart_;
  uint32_t sms_ = 148;
  unsigned pt_occ_ = 4;
  unsigned chi2_occ_ = 4;
  DBuf b_tmeta_, b_tcv_, b_taux_, b_tlin_, b_sspan_, b_runslot_;
  bool pipe_aux_pending_ = false;
  DBuf b_camtc_idx_, b_camtc_off_, b_dir_rb_, b_dir_re_;
  const uint64_t* dir_rbeg_ = nullptr;
  const uint64_t* dir_rend_ = nullptr;
  int dir_nranges_ = 0;
  unsigned dir_rest_grid_ = 1;
  DBuf b_cpre_, b_cpre_new_;
  DBuf b_J_, b_Rf_, b_w_, b_part_, b_x_, b_xn_, b_b_, b_cl_, b_D_, b_dx_, b_Hc_, b_Hp_, b_Mc_, b_Mp_, b_xs_, b_r_, b_z_, b_p_,
      b_ap_, b_tr_, b_tr2_, b_tf_, b_cr_, b_br_, b_br2_, b_bf_;
};

std::unique_ptr<SolverBase> make_solver(GraphData& g) {
  switch (g.precision) {
    case GB_FP64: return std::make_unique<Solver<double, double>>(g);
    case GB_FP32: return std::make_unique<Solver<float, float>>(g);
    case GB_FP32_BF16: return std::make_unique<Solver<float, bf16>>(g);
  }
  throw std::invalid_argument("invalid precision pair");
}

}  // namespace gb

// ======================================================================= C ABI
namespace {
thread_local std::string g_err;

int set_err(int code, const std::string& what) {
  g_err = what;
  return code;
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    g_err.clear();
    return GB_OK;
  } catch (const gb::NoDevice& e) {
    return set_err(GB_ERR_NO_DEVICE, e.what());
  } catch (const gb::CudaError& e) {
    return set_err(GB_ERR_CUDA, e.what());
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
}  // namespace

struct gb_graph {
  gb::GraphData data;
  std::unique_ptr<gb::SolverBase> solver;
  gb::SolverBase& get() {
    if (!solver) solver = gb::make_solver(data);
    return *solver;
  }
};

namespace gb {
// FMA throughput probe: 8 independent accumulator chains per thread, 2 blocks
// of 256 threads per SM, every SM busy.
template <typename T>
__global__ void k_fma_probe(T* out, int iters, T a, T b) {
  T x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = static_cast<T>(threadIdx.x + k);
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
  T s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == static_cast<T>(-1.2345)) out[0] = s;  // keeps the chains alive
}

}  // namespace gb

extern "C" {

void gb_default_config(gb_lm_config* c) {
  c->max_iterations = 10;
  c->tolerance = 1e-6;
  c->level = 0;
  c->tau = 1e-4;
  c->pcg.max_iterations = 50;
  c->pcg.tolerance = 1e-6;
  c->pcg.rejection_ratio = 10.0;
  c->pcg.normalize_rhs = 1;
  c->clamp_min = 1e-6;
  c->clamp_max = 1e32;
  c->damping = GB_DAMPING_AFTER_SCALING;
  c->use_rejection_guard = 1;
  c->refresh_on_reject = 0;
  c->lambda_max = 1e32;
  c->gradient_tolerance = 1e-12;
}

const char* gb_last_error(void) { return g_err.c_str(); }

int gb_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

gb_graph* gb_create(int precision, int diff_mode, int device) {
  gb_graph* out = nullptr;
  const int rc = guarded([&] {
    if (precision < GB_FP64 || precision > GB_FP32_BF16)
      throw std::invalid_argument("invalid precision pair");
    if (diff_mode < GB_ANALYTIC || diff_mode > GB_DYNAMIC) throw std::invalid_argument("unknown differentiation mode");
    const int n = gb_device_count();
    if (n == 0) throw gb::NoDevice("no CUDA device visible: the B200 solver has no CPU fallback");
    if (device < 0 || device >= n) throw std::invalid_argument("invalid CUDA device ordinal");
    auto* g = new gb_graph;
    g->data.precision = precision;
    g->data.diff_mode = diff_mode;
    g->data.device = device;
    out = g;
  });
  (void)rc;
  return out;
}

void gb_destroy(gb_graph* g) { delete g; }

int gb_set_cameras(gb_graph* g, void* params, uint64_t n, const uint8_t* fixed) {
  return guarded([&] {
    if (!params && n) throw std::invalid_argument("add_vertex: null handle");
    g->data.cams = params;
    g->data.nc = n;
    g->data.cam_fixed.assign(fixed ? fixed : nullptr, fixed ? fixed + n : nullptr);
    ++g->data.revision;
  });
}

int gb_set_points(gb_graph* g, void* params, uint64_t n, const uint8_t* fixed) {
  return guarded([&] {
    if (!params && n) throw std::invalid_argument("add_vertex: null handle");
    g->data.pts = params;
    g->data.np = n;
    g->data.pt_fixed.assign(fixed ? fixed : nullptr, fixed ? fixed + n : nullptr);
    ++g->data.revision;
  });
}

int gb_set_observations(gb_graph* g, uint64_t n, const uint32_t* cam, const uint32_t* pt, const void* observed,
                        const uint8_t* level, int loss_kind, double huber_delta) {
  return guarded([&] {
    gb::GraphData& d = g->data;
    if (n > 0xffffffffull) throw std::invalid_argument("more than 2^32 observations");
    if (loss_kind != GB_LOSS_DEFAULT && loss_kind != GB_LOSS_HUBER) throw std::invalid_argument("unknown loss kind");
    if (n && (!cam || !pt || !observed)) throw std::invalid_argument("null observation arrays");
    d.ne = n;
    d.cam_idx = cam;
    d.pt_idx = pt;
    if (d.precision == GB_FP64) {
      d.obs_conv.clear();
      d.obs = static_cast<const double*>(observed);
    } else {
      const float* o = static_cast<const float*>(observed);
      d.obs_conv.assign(o, o + 2 * n);
      d.obs = d.obs_conv.data();
    }
    d.level = level;
    d.loss_kind = loss_kind;
    d.huber = huber_delta;
    ++d.revision;
  });
}

int gb_set_linear_solver(gb_graph* g, int solver) {
  return guarded([&] {
    if (solver != GB_SOLVER_PCG && solver != GB_SOLVER_SCHUR) throw std::invalid_argument("unknown linear solver");
    g->data.linear_solver = solver;
    if (g->solver) g->solver.reset();
  });
}

int gb_set_differentiation_mode(gb_graph* g, int mode) {
  return guarded([&] {
    if (mode < GB_ANALYTIC || mode > GB_DYNAMIC) throw std::invalid_argument("unknown differentiation mode");
    if (mode != g->data.diff_mode) {
      g->data.diff_mode = mode;
      ++g->data.revision;
    }
  });
}

int gb_optimize(gb_graph* g, const gb_lm_config* cfg, gb_solve_report* report, gb_iteration_record* records,
                int32_t max_records) {
  return guarded([&] { g->get().optimize(*cfg, report, records, max_records); });
}

int gb_begin(gb_graph* g, const gb_lm_config* cfg, gb_solve_report* report) {
  return guarded([&] { g->get().begin(*cfg, report); });
}

int gb_step(gb_graph* g, int32_t n) {
  return guarded([&] { g->get().step(n); });
}

int gb_end(gb_graph* g, gb_solve_report* report, gb_iteration_record* records, int32_t max_records) {
  return guarded([&] { g->get().end(report, records, max_records); });
}

void* gb_stream(gb_graph* g) {
  void* s = nullptr;
  guarded([&] { s = g->get().stream(); });
  return s;
}

int gb_time_hvp(gb_graph* g, int32_t reps, double* ms_pair, double* ms_tiles) {
  return guarded([&] { g->get().time_hvp(reps < 1 ? 1 : reps, ms_pair, ms_tiles); });
}

int gb_iteration_kernels(gb_graph* g, int32_t* kernels) {
  return guarded([&] { *kernels = g->get().iteration_kernels(); });
}

int gb_hvp_bytes(gb_graph* g, double* kernel_bytes, double* reference_bytes) {
  return guarded([&] { g->get().hvp_bytes(kernel_bytes, reference_bytes); });
}

int gb_hvp_info(gb_graph* g, int32_t* path, double* kernel_bytes, double* algorithmic_bytes,
                double* algorithmic_flops) {
  return guarded([&] {
    g->get().hvp_bytes(kernel_bytes, nullptr);
    g->get().hvp_info(path, algorithmic_bytes, algorithmic_flops);
  });
}

int gb_fma_peak(int32_t device, int32_t precision, double* tflops) {
  using namespace gb;
  return guarded([&] {
    CK(cudaSetDevice(device));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    DBuf o;
    void* out = o.alloc(16);
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const int iters = 4096, blocks = 2 * sms, threads = 256;
    float ms = 0;
    for (int rep = 0; rep < 3; ++rep) {  // first pass warms the clocks
      CK(cudaEventRecord(e0));
      if (precision == 0)
        gb::k_fma_probe<double><<<blocks, threads>>>(static_cast<double*>(out), iters, 0.999999, 1e-7);
      else
        gb::k_fma_probe<float><<<blocks, threads>>>(static_cast<float*>(out), iters, 0.999999f, 1e-7f);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&ms, e0, e1));
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    const double flops = 2.0 * 8.0 * iters * static_cast<double>(blocks) * threads;
    if (tflops) *tflops = flops / (ms * 1e-3) / 1e12;
  });
}

void* gb_host_alloc(uint64_t bytes) { return gb::HostCache::get().alloc(static_cast<size_t>(bytes)); }

void gb_host_free(void* p) { gb::HostCache::get().release(p); }

void gb_host_copy(void* dst, const void* src, uint64_t bytes) {
  // large copies split over host threads (one thread moves ~10-15 GB/s)
  const uint64_t chunk = uint64_t(8) << 20;
  const unsigned hw = std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
  const unsigned nt = static_cast<unsigned>(std::min<uint64_t>(hw, (bytes + chunk - 1) / chunk));
  if (nt <= 1) {
    if (bytes) std::memcpy(dst, src, bytes);
    return;
  }
  const uint64_t per = (bytes + nt - 1) / nt;
  std::vector<std::thread> th;
  for (unsigned i = 0; i < nt; ++i) {
    const uint64_t lo = i * per, hi = std::min(bytes, lo + per);
    if (lo >= hi) break;
    th.emplace_back([=] { std::memcpy(static_cast<char*>(dst) + lo, static_cast<const char*>(src) + lo, hi - lo); });
  }
  for (auto& t : th) t.join();
}

int gb_nccl_unique_id(void* out128) {
  return guarded([&] { gb::nccl_unique_id(out128); });
}

int gb_shm_allreduce_selftest(int world, int rank, uint64_t key, double* data, uint64_t n, int max, double* bcast,
                              uint64_t nb) {
  return guarded([&] { gb::shm_allreduce_selftest(world, rank, key, data, n, max, bcast, nb); });
}

int gb_set_distributed(gb_graph* g, int world, int rank, int kind, const void* id) {
  return guarded([&] {
    if (world < 1) {
      g->data.reducer.reset();
    } else {
      if (cudaSetDevice(g->data.device) != cudaSuccess) throw gb::CudaError("cudaSetDevice failed");
      g->data.reducer = gb::make_reducer(kind, world, rank, id);
    }
    g->solver.reset();
    ++g->data.revision;
  });
}

int gb_shard_plan(uint64_t num_cameras, uint64_t num_points, uint64_t n, const uint32_t* camera_index,
                  const uint32_t* point_index, int world, uint32_t* tiles_out, uint32_t* points_out,
                  uint64_t* edges_out, uint32_t* point_owner) {
  return guarded([&] {
    gb::ActivationInput in;
    in.nc = num_cameras;
    in.np = num_points;
    in.ne = n;
    in.cam = camera_index;
    in.pt = point_index;
    gb::Activation full;
    gb::activate(in, full);
    for (int r = 0; r < world; ++r) {
      uint32_t t0, t1, p0, p1;
      gb::shard_range(full, world, r, &t0, &t1, &p0, &p1);
      tiles_out[2 * r] = t0;
      tiles_out[2 * r + 1] = t1;
      points_out[2 * r] = p0;
      points_out[2 * r + 1] = p1;
      uint64_t e = 0;
      for (uint32_t t = t0; t < t1; ++t) e += full.tile_ecnt[t];
      edges_out[r] = e;
      if (point_owner)
        for (uint32_t i = p0; i < p1; ++i) point_owner[full.pt_order[i]] = static_cast<uint32_t>(r);
    }
  });
}

int gb_activation_selfcheck(gb_graph* g, int level) {
  return guarded([&] {
    const std::string e = g->get().selfcheck(level);
    if (!e.empty()) throw std::logic_error("device activation differs from host activation: " + e);
  });
}

int gb_mse(gb_graph* g, double* out) {
  return guarded([&] {
    if (g->data.ne == 0) {
      *out = 0.0;
      return;
    }
    *out = g->get().residual_sum(0, true) / static_cast<double>(g->data.ne);
  });
}

int gb_total_error(gb_graph* g, int level, double* out) {
  return guarded([&] { *out = g->get().residual_sum(level, false); });
}

int gb_ls_linearize(gb_graph* g, int level, double cmin, double cmax, int damping, double* chi2, int64_t* n, void* b,
                    void* diag, void* clamped, void* scaling, int32_t* finite) {
  return guarded([&] { g->get().ls_linearize(level, cmin, cmax, damping, chi2, n, b, diag, clamped, scaling, finite); });
}

int gb_ls_hvp(gb_graph* g, const void* v, void* out, double lambda) {
  return guarded([&] { g->get().ls_hvp(v, out, lambda); });
}

int gb_ls_preconditioner(gb_graph* g, double lambda, void* blocks, int32_t* fallbacks) {
  return guarded([&] { g->get().ls_precond(lambda, blocks, fallbacks); });
}

int gb_ls_solve_step(gb_graph* g, double lambda, const gb_pcg_config* pcg, void* dx, gb_pcg_stats* stats, double* pred,
                     int32_t* finite) {
  return guarded([&] { g->get().ls_solve_step(lambda, *pcg, dx, stats, pred, finite); });
}

int gb_ls_jacobians(gb_graph* g, void* out) {
  return guarded([&] { g->get().ls_jacobians(out); });
}

int gb_incidence(gb_graph* g, int descriptor, uint64_t* nseg, uint64_t* nitems, uint64_t* vos, uint64_t* offsets,
                 uint32_t* items_factor, uint16_t* items_slot) {
  return guarded([&] {
    if (descriptor != 0 && descriptor != 1) throw std::out_of_range("incidence index");
    const gb::Activation& a = g->get().activation();
    const gb::Incidence& inc = descriptor == 0 ? a.cam_inc : a.pt_inc;
    if (nseg) *nseg = inc.vertex_of_segment.size();
    if (nitems) *nitems = inc.items.size();
    if (vos) std::copy(inc.vertex_of_segment.begin(), inc.vertex_of_segment.end(), vos);
    if (offsets) std::copy(inc.offsets.begin(), inc.offsets.end(), offsets);
    if (items_factor) std::copy(inc.items.begin(), inc.items.end(), items_factor);
    if (items_slot) std::fill(items_slot, items_slot + inc.items.size(), static_cast<uint16_t>(descriptor));
  });
}

}  // extern "C"
