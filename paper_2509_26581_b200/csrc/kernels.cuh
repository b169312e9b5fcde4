// Device kernels of the LM inner loop. See DESIGN.md for the data layout and
// the roofline of each kernel. Reference semantics are cited per kernel.
//
// Layout recap (all device-resident for the whole solve):
//   columns   internal layout: camera c at [9c, 9c+9) (insertion order),
//             point i (internal order) at [9nc + 3i, 9nc + 3i + 3). Fixed
//             vertices keep their columns but every vector is 0 there, so
//             dot products and norms equal the reference's free-only ones.
//   edges     "device order" d: point tiles (<= kTileEdges edges, <=
//             kTilePoints points), inside a tile sorted by (camera, factor).
//             SoA: cam[d], lpt[d], obs[2][d], J[24][d] (SP, row-major Jc|Jp).
//   cameras   per-warp-chunk camera runs are reduced with shuffles and
//             written to partial slots; a camera kernel sums its slots in
//             slot order (deterministic, no float atomics).
//   points    per-edge point contributions are staged in shared memory and
//             summed per point in slot order inside the tile.
#pragma once

#include <cooperative_groups.h>
#include <utility>

#include "activate.hpp"
#include "common.cuh"
#include "gb_bal.h"
#include "snavely.cuh"

namespace gb {

// packed upper-triangular (row-major, i <= j) index helpers; always called
// with compile-time arguments inside unrolled loops so register arrays stay
// in registers.
__host__ __device__ constexpr int p9row(int q) {
  int i = 0;
  while (q >= 9 - i) {
    q -= 9 - i;
    ++i;
  }
  return i;
}
__host__ __device__ constexpr int p9col(int q) {
  int i = 0;
  while (q >= 9 - i) {
    q -= 9 - i;
    ++i;
  }
  return i + q;
}
// std::clamp semantics (NaN passes through), linear_system.hpp:75
template <typename T>
__host__ __device__ inline T clampv(T v, T lo, T hi) {
  return v < lo ? lo : (hi < v ? hi : v);
}
__host__ __device__ constexpr int p9(int i, int j) { return i <= j ? i * 9 - i * (i - 1) / 2 + (j - i) : j * 9 - j * (j - 1) / 2 + (i - j); }
__host__ __device__ constexpr int p3(int i, int j) { return i <= j ? i * 3 - i * (i - 1) / 2 + (j - i) : j * 3 - j * (j - 1) / 2 + (i - j); }

constexpr int kLinVals = 54;  // per camera run at linearize: b (9) + upper H (45)
constexpr int kGsStride = kTileThreads + 4;  // row stride of the HVP camera-value staging (bank spread)
constexpr int kCamWarps = 8;  // warps per block in camera kernels

// Device-resident solver state (one per handle). Scalars are FP like the
// reference's locals (levenberg_marquardt.hpp:145-147, pcg.hpp:303-330).
template <typename FP>
struct State {
  // configuration
  double tol, grad_tol, lambda_max, tau, pcg_tol, pcg_ratio;
  double clamp_min, clamp_max;
  int max_iterations, pcg_max_it, normalize_rhs, before_scaling, use_guard, refresh_on_reject;
  int schur;  // linear solver: 0 full-system PCG (reference), 1 Schur complement on the cameras
  // PCG
  FP rho, pap, alpha, beta, rhs_norm, scale, unscale, ref_norm;
  double pcg_relres;
  int pcg_it, pcg_done, pcg_conv, pcg_zero;
  int dir_pending;  // p = z + beta p still to be applied to normal-tile points (fused into k_hvp_pipe)
  int x_pending;    // x += alpha p of the last PCG update still to be applied (defer_x: by the next HVP or k_step)
  // step / candidate
  FP pred, chi2_new;
  int step_finite;
  // LM
  FP chi2, lambda, nu, lambda_solve, rel_decrease;
  int lm_it, terminated, termination, iter_active, accepted, do_linearize, accepted_steps, fallbacks;
  // linearization
  FP lin_chi2, grad_max;
  int lin_finite;
  // last-block counters, one per kernel that uses them
  unsigned cnt[16];
};

template <typename FP, typename SP>
struct Dev {
  using A = arith_t<SP>;
  uint32_t nc, np, na, ntiles, nparts;  // na = padded edge slots (row stride of J, obs, w)
  uint64_t ncols;  // 9nc + 3np
  FP* x;
  FP* x_new;
  const uint8_t* col_free;  // ncols
  const uint32_t* d_cam;
  const uint16_t* d_lpt;
  const FP* d_obs;  // [2][na]
  SP* J;            // [24][na] full store, [16][na] factored store (jfact), or null (dynamic)
  FP* Rf;           // [nc][10] factored store: R (row-major 3x3) and f per camera
  FP* cpre;         // [nc][kCamPre] per-camera chain record at x (snavely.cuh camera_pre)
  FP* cpre_new;     // [nc][kCamPre] at the chi^2 evaluation point
  int jfact;        // 1: factored J store (analytic mode, SP == FP), DESIGN.md §2
  int want_dx;      // k_step also stores dx (the LinearSystem::solve_step surface only)
  int defer_x;      // recompute path: k_pcg_update leaves x += alpha p to the next HVP (its loader reads p anyway)
  // pipelined HVP (hvp_pipe.cuh): tile records and per-tile camera copies
  const uint32_t* tile_meta;  // [n_normal][12] (hvp_pipe.cuh TileMeta)
  uint32_t ntcams;            // tile_cam_off[ntiles]
  arith_t<SP>* tcv;           // [ntcams][9]  D*p of each tile's cameras
  unsigned char* tile_aux;    // static per-tile blobs (hvp_pipe.cuh AuxSec)
  uint2* slot_span;           // [nparts] per run: tile-relative edge range [lo, hi) (lo | hi << 16), storage slot
  const uint32_t* run_slot;   // [nparts] run (chunk_part_base + r) -> storage slot: camera-major, so each
                              // camera's partials are contiguous for the camera kernels (position in cam_part_idx)
  unsigned char* tile_lin;    // per-linearization per-tile blobs (LinSec)
  const uint32_t* cam_tc_off;  // [nc+1] camera -> its tile-camera entries (tcv rows)
  const uint32_t* cam_tc_idx;
  // recompute HVP (hvp_rc.cuh): per-camera HVP records, per tile-camera
  // 15-value partials, heavy-tile partial-slot flags
  FP* crec;              // [nc][16]
  FP* part15;            // [ntcams][16]
  const uint8_t* hflag;  // [nparts] camera-major storage order
  FP* lpart;             // [ntcams][54] linearize camera-run sums of normal tiles (k_lin_seg), or null
  FP* w;            // [na] or null (default loss: w == 1)
  const uint32_t* tile_ebeg;  // padded slot begin of each tile
  const uint32_t* tile_ecnt;  // real edges of each tile
  const uint32_t* tile_pbeg;
  const uint16_t* d_lcam;        // local camera index (normal tiles)
  const uint32_t* tile_cam_off;  // distinct cameras of each tile
  const uint32_t* tile_cams;
  const uint32_t* normal_tiles;
  const uint32_t* heavy_tiles;
  uint32_t n_normal, n_heavy;
  const uint32_t* tile_chunk_base;
  const uint32_t* chunk_part_base;
  const uint32_t* pt_slot_off;
  const uint16_t* pt_slots;
  const uint32_t* cam_part_off;
  const uint32_t* cam_part_idx;
  FP* part;  // [nparts][54]
  FP* b;
  FP* clamped;
  FP* D;
  FP* Hc;  // [nc][45]
  FP* Hp;  // [np][6]
  FP* Mc;  // [nc][45]
  FP* Mp;  // [np][6]
  SP* xs;
  SP* r;
  SP* z;
  SP* p;
  SP* ap;
  A* vt;       // (Arith) D * p for every column, refreshed with p (HVP gather source)
  FP* rc;      // Schur: reduced camera rhs (9nc)
  FP* xp;      // Schur: back-substituted point step (3np), unscaled
  A* dbg_out;  // optional wide HVP output (LinearSystem::hvp surface)
  FP* dx;
  FP* tile_red;   // [ntiles * 8] (HVP: one dot partial per warp of a tile)
  FP* tile_red2;  // [ntiles]
  int* tile_flag; // [ntiles]
  FP* cam_red;    // [nc]
  FP* blk_red;    // [nblk]
  FP* blk_red2;   // [nblk]
  int* blk_flag;  // [nblk]
  State<FP>* st;
  gb_iteration_record* recs;
  int loss_kind;
  FP huber;
  // sharding: world ranks own disjoint point tiles; cameras
  // are replicated and counted in dot products on rank 0 only. world > 1:
  // every reduction site writes a per-rank partial into red/redmax, the host
  // allreduces it, and a finalize kernel applies the decision.
  int world, rank, dist;  // dist: a reducer is attached (even with world == 1)
  FP* red;     // SUM partials (layout: kRed* below)
  FP* redmax;  // MAX partials
};

// red layout: [0, 54 nc) camera sums (linearize b+H / HVP J^T q), then scalars
template <typename FP, typename SP>
__host__ __device__ inline uint64_t red_scalars(const Dev<FP, SP>& d) {
  return 54ull * d.nc + 8;
}
enum RedSlot : int {
  kRedLinChi = 0, kRedLinFail, kRedDampAny, kRedRhs, kRedFallback, kRedInitRz, kRedInitRr, kRedHvpDot,
  kRedUpdRz, kRedUpdRr, kRedStepPred, kRedStepFail, kRedChi, kRedCount
};
enum RedMaxSlot : int { kRedMaxLin = 0, kRedMaxDamp, kRedMaxCount };

// columns counted in dot products / norms on this rank (cameras: rank 0 only)
template <typename FP, typename SP>
__device__ inline bool counted(const Dev<FP, SP>& d, uint64_t col) {
  return d.rank == 0 || col >= 9ull * d.nc;
}

// ---- decisions, shared by the fused last blocks (world == 1) and the
// finalize kernels (world > 1)
template <typename FP>
__device__ inline void fin_lin(State<FP>* st, FP chi, bool all_finite, FP gmax) {
  st->lin_chi2 = chi;
  st->grad_max = fmax(gmax, FP(0));
  st->lin_finite = (all_finite && is_finite(chi)) ? 1 : 0;
}
template <typename FP>
__device__ inline void fin_damp(State<FP>* st, FP m, bool any) {
  const FP tau = static_cast<FP>(st->tau);
  st->lambda = any ? tau * fmax(m, FP(0)) : tau;
  st->nu = FP(2);
}
template <typename FP>
__device__ inline void fin_rhs(State<FP>* st, FP s) {  // pcg.hpp:303-311
  const FP nrm = sqrt(s);
  st->rhs_norm = nrm;
  if (!(nrm > FP(0))) {
    st->pcg_done = 1;
    st->pcg_zero = 1;
    st->pcg_conv = is_finite(nrm) ? 1 : 0;
    st->pcg_relres = 0.0;
  }
  st->scale = st->normalize_rhs ? FP(1) / nrm : FP(1);
  st->ref_norm = st->normalize_rhs ? FP(1) : nrm;
  st->unscale = st->normalize_rhs ? nrm : FP(1);
}
template <typename FP>
__device__ inline void fin_init(State<FP>* st, FP rz, FP rr) {  // pcg.hpp:326-329
  if (!st->pcg_done) {
    st->rho = rz;
    st->pcg_relres = static_cast<double>(sqrt(rr) / st->ref_norm);
  }
}
template <typename FP>
__device__ inline void fin_hvp(State<FP>* st, FP pap) {  // pcg.hpp:334-340
  st->pap = pap;
  if (!(pap > FP(0)) || !is_finite(pap)) {
    st->pcg_done = 1;
    st->pcg_conv = 0;
  } else {
    st->alpha = st->rho / pap;
  }
}
template <typename FP>
__device__ inline void fin_upd(State<FP>* st, FP rz, FP rr) {  // pcg.hpp:345-359
  st->pcg_it += 1;
  const FP res = sqrt(rr);
  const double rel = static_cast<double>(res / st->ref_norm);
  st->pcg_relres = rel;
  if (!isfinite(rel)) {
    st->pcg_done = 1;
    st->pcg_conv = 0;
  } else if (res <= static_cast<FP>(st->pcg_tol) * st->ref_norm) {
    st->pcg_done = 1;
    st->pcg_conv = 1;
  } else {
    st->beta = rz / st->rho;
    st->rho = rz;
  }
}
template <typename FP>
__device__ inline void fin_step(State<FP>* st, FP pred, bool finite) {
  st->pred = pred;
  st->step_finite = finite ? 1 : 0;
}


// ------------------------------------------------------------------ helpers

// Warp-segmented suffix reduction over runs of equal camera inside a warp
// chunk: afterwards the head lane of each run holds the run total. Fixed
// association order (deterministic). run_end: last lane of this lane's run.
template <typename T, int K>
__device__ inline void seg_reduce(T (&v)[K], int lane, int run_end) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const T t = __shfl_down_sync(0xffffffffu, v[k], o);
      if (lane + o <= run_end) v[k] += t;
    }
  }
}

// run_slot[cam_part_idx[q]] = q: partial-slot storage in camera-list order
static __global__ void k_run_slots(uint32_t n, const uint32_t* cam_part_idx, uint32_t* run_slot) {
  for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x)
    run_slot[cam_part_idx[q]] = q;
}

// Sum of src[lo, hi) in a fixed association order (4 interleaved partial
// sums), stored to *dst. Every camera-run reduction of the HVP goes through it,
// so the tile kernels and the pipelined kernel produce identical bits.
template <typename A, typename FP>
__device__ __forceinline__ void run_sum_store(const A* src, uint32_t lo, uint32_t hi, FP* dst) {
  A a0 = A(0), a1 = A(0), a2 = A(0), a3 = A(0);
  uint32_t e = lo;
  for (; e + 4 <= hi; e += 4) {
    a0 += src[e];
    a1 += src[e + 1];
    a2 += src[e + 2];
    a3 += src[e + 3];
  }
  for (; e < hi; ++e) a0 += src[e];
  *dst = static_cast<FP>((a0 + a1) + (a2 + a3));
}

// Camera-run sums of a warp chunk from shared memory: the chunk's 32 edges
// have written their 9 camera values to gw[k * stride + lane]; lane o of the
// warp produces output o = 9 r + k (run r, value k) as a sequential sum over
// the run's edges, so the 9R outputs of a chunk with R runs are plain loads
// and adds (no shuffle trees) and their slot writes are contiguous. Fixed
// association order (deterministic). heads/vm: ballots of run heads / valid lanes.
template <typename A, typename FP>
__device__ inline void chunk_runs_smem(const A* gw, int stride, int lane, unsigned heads, unsigned vm,
                                       uint32_t slot0, FP* part, const uint32_t* run_slot) {
  const int R = __popc(heads);
  const int end = 32 - __clz(vm);
  // lane q holds start(q) = the q-th head (run q spans [start(q), start(q + 1)))
  int my_start = end;
  {
    unsigned hs = heads;
    for (int k = 0; hs; ++k) {
      const int pos = __ffs(hs) - 1;
      hs &= hs - 1;
      if (lane == k) my_start = pos;
    }
  }
  for (int base = 0; base < 9 * R; base += 32) {  // warp-uniform passes
    const int o = base + lane;
    const int r = min((o * 57) >> 9, 31);  // o / 9 for o < 512
    const int k = o - 9 * r;
    const int start = __shfl_sync(0xffffffffu, my_start, r);
    const int nxt = __shfl_sync(0xffffffffu, my_start, min(r + 1, 31));
    if (o >= 9 * R) continue;
    const int stp = r + 1 < R ? nxt : end;
    run_sum_store<A, FP>(gw + k * stride, start, stp, part + static_cast<uint64_t>(run_slot[slot0 + r]) * 9 + k);
  }
}

// Camera-run sums of one warp chunk (k_hvp_tiles): the chunk's edges stage
// their 9 camera values in shared memory and chunk_runs_smem sums each run in
// run_sum_store order, the order k_hvp_pipe uses tile-wide (identical bits).
template <typename A, typename FP>
__device__ inline void camera_runs(const A (&g)[9], int lane, unsigned hm, unsigned vm, uint32_t slot0, A* gw,
                                   int stride, FP* part, const uint32_t* run_slot) {
  if (!hm) return;
#pragma unroll
  for (int k = 0; k < 9; ++k) gw[k * stride + lane] = g[k];
  __syncwarp();
  chunk_runs_smem<A, FP>(gw, stride, lane, hm, vm, slot0, part, run_slot);
  __syncwarp();
}

struct RunInfo {
  bool head;
  int run_end;
  uint32_t slot;
};

__device__ inline RunInfo run_info(uint32_t cam, bool valid, uint32_t chunk_slot_base) {
  const int lane = threadIdx.x & 31;
  const uint32_t prev = __shfl_up_sync(0xffffffffu, cam, 1);
  const bool head = valid && (lane == 0 || cam != prev);
  const unsigned hm = __ballot_sync(0xffffffffu, head);
  const unsigned vm = __ballot_sync(0xffffffffu, valid);
  const unsigned later = lane == 31 ? 0u : (hm & (0xffffffffu << (lane + 1)));
  RunInfo ri;
  ri.head = head;
  ri.run_end = later ? (__ffs(later) - 2) : (vm ? 31 - __clz(vm) : -1);
  ri.slot = chunk_slot_base + __popc(hm & ((1u << lane) - 1u));
  return ri;
}

// Factored J store (analytic mode with SP == FP): per edge 16
// rows [Jc(:,0:3) row 0 | row 1 | U = du/dP (2x3) | dist | n | p0 | p1];
// per camera Rf = [R | f]. The rebuilt entries are bit-identical to the
// chain's (same explicitly rounded operations, snavely.cuh), so the stored
// operator is exactly J; it moves 16 instead of 24 values per edge.
constexpr int kJFactRows = 16;

// J store layout: blocks of kJBlock slots (a normal tile is exactly one block,
// so the pipelined HVP moves it with ONE bulk copy); inside a block, row k of
// the tile's J at a padded row stride (16 bytes of padding spread the shared-
// memory banks of the HVP's contribution rows that overlay it).
template <typename SP>
__host__ __device__ constexpr int jstore_stride() {
  return static_cast<int>((kJBlock * sizeof(SP) + 16) / sizeof(SP));
}
template <typename SP>
__host__ __device__ inline uint64_t jidx(uint32_t e, int k, int rows) {
  static_assert(kJBlock == 512, "block index by shift");
  return static_cast<uint64_t>(e >> 9) * (static_cast<uint64_t>(rows) * jstore_stride<SP>()) +
         static_cast<uint64_t>(k) * jstore_stride<SP>() + (e & 511u);
}
// elements of the J store for ns slots (a multiple of kJBlock)
template <typename SP>
__host__ __device__ inline uint64_t jstore_elems(uint64_t ns, int rows) {
  return (ns + kJBlock - 1) / kJBlock * static_cast<uint64_t>(rows) * jstore_stride<SP>();
}

template <typename FP, typename SP>
__device__ inline void store_J(const Dev<FP, SP>& d, uint32_t e, const FP* jc, const FP* jp, const FP* fac) {
  if (d.jfact) {
    constexpr int R = kJFactRows;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      d.J[jidx<SP>(e, k, R)] = narrow<SP>(jc[k]);
      d.J[jidx<SP>(e, 3 + k, R)] = narrow<SP>(jc[9 + k]);
    }
#pragma unroll
    for (int k = 0; k < 10; ++k) d.J[jidx<SP>(e, 6 + k, R)] = narrow<SP>(fac[k]);
  } else {
#pragma unroll
    for (int k = 0; k < 18; ++k) d.J[jidx<SP>(e, k, 24)] = narrow<SP>(jc[k]);
#pragma unroll
    for (int k = 0; k < 6; ++k) d.J[jidx<SP>(e, 18 + k, 24)] = narrow<SP>(jp[k]);
  }
}

template <typename FP, typename SP>
__device__ inline void load_J(const Dev<FP, SP>& d, uint32_t e, uint32_t cam, arith_t<SP>* jc, arith_t<SP>* jp) {
  using A = arith_t<SP>;
  const SP* J = d.J;
  if constexpr (std::is_same<SP, FP>::value) {
    if (d.jfact) {
      constexpr int RR = kJFactRows;
      FP U[6], R[9];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        jc[k] = J[jidx<SP>(e, k, RR)];
        jc[9 + k] = J[jidx<SP>(e, 3 + k, RR)];
      }
#pragma unroll
      for (int k = 0; k < 6; ++k) U[k] = J[jidx<SP>(e, 6 + k, RR)];
      const FP dist = J[jidx<SP>(e, 12, RR)], n = J[jidx<SP>(e, 13, RR)];
      const FP p0 = J[jidx<SP>(e, 14, RR)], p1 = J[jidx<SP>(e, 15, RR)];
      const FP* rf = d.Rf + 10ull * cam;
#pragma unroll
      for (int k = 0; k < 9; ++k) R[k] = rf[k];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        jc[3 + k] = U[k];
        jc[12 + k] = U[3 + k];
      }
      point_block<FP>(U, R, jp);
      intrinsic_cols<FP>(dist, n, p0, p1, rf[9], jc);
      return;
    }
  }
#pragma unroll
  for (int k = 0; k < 18; ++k) jc[k] = widen<A>(J[jidx<SP>(e, k, 24)]);
#pragma unroll
  for (int k = 0; k < 6; ++k) jp[k] = widen<A>(J[jidx<SP>(e, 18 + k, 24)]);
}

// Full 24-value rows from either store (LinearSystem accessor surface).
template <typename FP, typename SP>
__global__ void k_expand_J(Dev<FP, SP> d, SP* out) {
  using A = arith_t<SP>;
  for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < d.na;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    A jc[18], jp[6];
    load_J(d, static_cast<uint32_t>(e), d.d_cam[e], jc, jp);
#pragma unroll
    for (int k = 0; k < 18; ++k) out[k * static_cast<uint64_t>(d.na) + e] = narrow<SP>(jc[k]);
#pragma unroll
    for (int k = 0; k < 6; ++k) out[(18 + k) * static_cast<uint64_t>(d.na) + e] = narrow<SP>(jp[k]);
  }
}

// =====================================================================
// Linearize (FactorDescriptor::linearize factor_descriptor.hpp:272-292,
// accumulate_gradient_and_diagonal :322-370 and the unscaled half of
// accumulate_precond_blocks :435-482; LinearSystem::linearize
// linear_system.hpp:67-82). One CTA per tile: Snavely residual + both
// Jacobian blocks from one chain per edge, J narrowed to SP and stored SoA,
// camera b/H via warp-segmented runs -> partial slots, point b/H summed in
// shared memory. Point epilogue: clamp, D = 1/sqrt(clamped), finiteness,
// max |b|.
// =====================================================================
// Per-camera chain records (snavely.cuh camera_pre) of `params` into out.
// mode 0: for a linearization (runs when it does); 1: for the candidate chi^2
// (runs when k_chi2_tiles does); 2: unconditionally.
template <typename FP, typename SP>
__global__ void k_cam_pre(Dev<FP, SP> d, const FP* params, FP* out, int mode, int force) {
  if (mode == 0 && !force && !d.st->do_linearize) return;
  if (mode == 1 && !force && (!d.st->iter_active || !d.st->step_finite)) return;
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < d.nc; c += gridDim.x * blockDim.x) {
    FP cp[9], pre[kCamPre];
#pragma unroll
    for (int k = 0; k < 9; ++k) cp[k] = params[9ull * c + k];
    camera_pre<FP>(cp, pre);
#pragma unroll
    for (int k = 0; k < kCamPre; ++k) out[static_cast<uint64_t>(kCamPre) * c + k] = pre[k];
  }
}

template <typename FP, typename SP, bool STORE, bool AUTO>
__global__ void __launch_bounds__(kTileThreads) k_lin_tiles(Dev<FP, SP> d, const uint32_t* list, int force) {
  if (!force && !d.st->do_linearize) return;
  const uint32_t t = list ? list[blockIdx.x] : blockIdx.x;
  const uint32_t eb = d.tile_ebeg[t];
  const uint32_t pb = d.tile_pbeg[t], pe = d.tile_pbeg[t + 1];
  const uint32_t ne_t = d.tile_ecnt[t], npt = pe - pb;
  const bool heavy = ne_t > static_cast<uint32_t>(kTileEdges);
  const int tid = threadIdx.x, lane = tid & 31;
  const uint64_t pcol0 = 9ull * d.nc;

  __shared__ FP sX[kTilePoints * 3];
  __shared__ FP stage[kTileEdges * 9];
  __shared__ FP hacc[9];
  __shared__ FP scratch[32];

  for (uint32_t i = tid; i < npt * 3; i += blockDim.x) sX[i] = d.x[pcol0 + 3ull * pb + i];
  if (tid < 9) hacc[tid] = FP(0);
  __syncthreads();

  const int loss = d.loss_kind;
  const FP delta = d.huber;
  FP chi = FP(0);
  for (uint32_t c0 = 0; c0 < ne_t; c0 += kTileThreads) {
    const uint32_t j = c0 + tid;
    const bool valid = j < ne_t;
    const uint32_t e = eb + (valid ? j : 0);
    const uint32_t cam = d.d_cam[e];
    const uint32_t lp = d.d_lpt[e];
    FP cp[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) cp[k] = d.x[9ull * cam + k];
    const FP* X = &sX[3 * lp];
    FP res[2], jc[18], jp[6], fac[10];
    if (AUTO) {
      snavely_residual<FP>(cp, X, d.d_obs[e], d.d_obs[static_cast<uint64_t>(d.na) + e], res);
      snavely_jacobians_auto<FP>(cp, X, jc, jp);
    } else {
      snavely_linearize<FP>(cp, X, d.d_obs[e], d.d_obs[static_cast<uint64_t>(d.na) + e], res, jc, jp, fac,
                            d.cpre + static_cast<uint64_t>(kCamPre) * cam);
    }
    const FP s = res[0] * res[0] + res[1] * res[1];
    const FP w = valid ? loss_weight<FP>(loss, delta, s) : FP(0);
    if (valid) chi += loss_value<FP>(loss, delta, s);
    if (STORE) {
      if (valid) store_J(d, e, jc, jp, fac);
#pragma unroll
      for (int k = 0; k < 18; ++k) jc[k] = widen<FP>(narrow<SP>(jc[k]));
#pragma unroll
      for (int k = 0; k < 6; ++k) jp[k] = widen<FP>(narrow<SP>(jp[k]));
    }
    if (d.w && valid) d.w[e] = w;
    const FP wr0 = w * res[0], wr1 = w * res[1];
    if (!valid) {
#pragma unroll
      for (int k = 0; k < 18; ++k) jc[k] = FP(0);
#pragma unroll
      for (int k = 0; k < 6; ++k) jp[k] = FP(0);
    }
    // camera side: 6 groups of 9 values (b, then packed upper H)
    const uint32_t chunk = d.tile_chunk_base[t] + (c0 + (tid & ~31)) / 32;
    const RunInfo ri = run_info(cam, valid, d.chunk_part_base[chunk]);
#pragma unroll
    for (int g = 0; g < 6; ++g) {
      FP v[9];
#pragma unroll
      for (int k = 0; k < 9; ++k) {
        const int idx = 9 * g + k;
        if (idx < 9) {
          v[k] = jc[k] * (valid ? wr0 : FP(0)) + jc[9 + k] * (valid ? wr1 : FP(0));
        } else {
          const int q = idx - 9;
          const int a = p9row(q), bb = p9col(q);
          v[k] = w * (jc[a] * jc[bb] + jc[9 + a] * jc[9 + bb]);
        }
      }
      seg_reduce<FP, 9>(v, lane, ri.run_end);
      if (ri.head) {
        FP* dst = d.part + static_cast<uint64_t>(d.run_slot[ri.slot]) * kLinVals + 9 * g;
#pragma unroll
        for (int k = 0; k < 9; ++k) dst[k] = v[k];
      }
    }
    // point side: b (3) + packed H (6)
    FP pv[9];
    pv[0] = jp[0] * wr0 + jp[3] * wr1;
    pv[1] = jp[1] * wr0 + jp[4] * wr1;
    pv[2] = jp[2] * wr0 + jp[5] * wr1;
    pv[3] = w * (jp[0] * jp[0] + jp[3] * jp[3]);
    pv[4] = w * (jp[0] * jp[1] + jp[3] * jp[4]);
    pv[5] = w * (jp[0] * jp[2] + jp[3] * jp[5]);
    pv[6] = w * (jp[1] * jp[1] + jp[4] * jp[4]);
    pv[7] = w * (jp[1] * jp[2] + jp[4] * jp[5]);
    pv[8] = w * (jp[2] * jp[2] + jp[5] * jp[5]);
    if (!heavy) {
      if (valid)
#pragma unroll
        for (int k = 0; k < 9; ++k) stage[j * 9 + k] = pv[k];
    } else {
#pragma unroll
      for (int k = 0; k < 9; ++k) stage[tid * 9 + k] = valid ? pv[k] : FP(0);
      __syncthreads();
      if (tid < 9) {
        FP acc = hacc[tid];
        const uint32_t nvalid = min(static_cast<uint32_t>(kTileThreads), ne_t - c0);
        for (uint32_t q = 0; q < nvalid; ++q) acc += stage[q * 9 + tid];
        hacc[tid] = acc;
      }
      __syncthreads();
    }
  }
  __syncthreads();

  // point epilogue
  FP gmax = FP(0);
  int fin = 1;
  for (uint32_t i = tid; i < npt; i += blockDim.x) {
    FP acc[9];
    if (heavy) {
#pragma unroll
      for (int k = 0; k < 9; ++k) acc[k] = hacc[k];
    } else {
#pragma unroll
      for (int k = 0; k < 9; ++k) acc[k] = FP(0);
      for (uint32_t q = d.pt_slot_off[pb + i]; q < d.pt_slot_off[pb + i + 1]; ++q) {
        const uint32_t sl = d.pt_slots[q];
#pragma unroll
        for (int k = 0; k < 9; ++k) acc[k] += stage[sl * 9 + k];
      }
    }
    const uint64_t col = pcol0 + 3ull * (pb + i);
    const bool freev = d.col_free[col];
    const uint64_t pidx = static_cast<uint64_t>(pb + i);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const FP bk = freev ? acc[k] : FP(0);
      d.b[col + k] = bk;
      const FP diag = freev ? acc[3 + p3(k, k)] : FP(0);
      const FP cl = clampv(diag, FP(d.st->clamp_min), FP(d.st->clamp_max));
      d.clamped[col + k] = freev ? cl : FP(0);
      d.D[col + k] = freev ? FP(1) / sqrt(cl) : FP(0);
      if (freev) {
        fin &= (is_finite(bk) && is_finite(diag)) ? 1 : 0;
        gmax = fmax(gmax, fabs(bk));
      }
    }
#pragma unroll
    for (int k = 0; k < 6; ++k) d.Hp[6 * pidx + k] = freev ? acc[3 + k] : FP(0);
  }
  const FP tchi = block_sum(chi, scratch);
  const FP tmax = block_max(gmax, scratch);
  const int tfin = __syncthreads_and(fin);
  if (tid == 0) {
    d.tile_red[t] = tchi;
    d.tile_red2[t] = tmax;
    d.tile_flag[t] = tfin;
  }
}

// Camera side of the linearization: sum each camera's partial slots (slot
// order), write b_c, packed H_c, clamped diagonal and D; the last block
// finalizes chi^2, finiteness and max |b| (linear_system.hpp:67-90).
// phase 0: fused (world == 1); phase 1: per-rank camera sums and tile
// scalars into red/redmax; phase 2: camera b/H/D from the allreduced sums and
// the finalize.
// Sum of camera c's 54-value linearize partials in slot-list order (lane v:
// value v in a0, value 32 + v in a1); eight slots' loads in flight at a time.
// With lpart (recompute path): the camera's tile-camera entries (cam_tc order),
// then the flagged partial slots of heavy tiles.
template <typename FP, typename SP>
__device__ inline void lin_cam_sum(const Dev<FP, SP>& d, uint32_t c, int lane, FP& a0, FP& a1) {
  constexpr int B = 8;
  if (d.lpart) {
    const uint32_t beg = d.cam_tc_off[c], end = d.cam_tc_off[c + 1];
    for (uint32_t q0 = beg; q0 < end; q0 += B) {
      const uint32_t mine = q0 + (lane & (B - 1)) < end ? d.cam_tc_idx[q0 + (lane & (B - 1))] : 0u;
      FP v0[B], v1[B];
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const FP* src = d.lpart + static_cast<uint64_t>(__shfl_sync(0xffffffffu, mine, u)) * kLinVals;
        const bool ok = q0 + u < end;
        v0[u] = ok ? src[lane] : FP(0);
        v1[u] = ok && lane < kLinVals - 32 ? src[32 + lane] : FP(0);
      }
#pragma unroll
      for (int u = 0; u < B; ++u)
        if (q0 + u < end) {
          a0 += v0[u];
          a1 += v1[u];
        }
    }
    if (d.n_heavy)
      for (uint32_t q = d.cam_part_off[c]; q < d.cam_part_off[c + 1]; ++q)
        if (d.hflag[q]) {
          a0 += d.part[static_cast<uint64_t>(q) * kLinVals + lane];
          if (lane < kLinVals - 32) a1 += d.part[static_cast<uint64_t>(q) * kLinVals + 32 + lane];
        }
    return;
  }
  const uint32_t beg = d.cam_part_off[c], end = d.cam_part_off[c + 1];
  for (uint32_t q0 = beg; q0 < end; q0 += B) {
    const uint32_t mine = q0 + (lane & (B - 1)) < end ? q0 + (lane & (B - 1)) : 0u;  // storage slot = position
    FP v0[B], v1[B];
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const FP* src = d.part + static_cast<uint64_t>(__shfl_sync(0xffffffffu, mine, u)) * kLinVals;
      const bool ok = q0 + u < end;
      v0[u] = ok ? src[lane] : FP(0);
      v1[u] = ok && lane < kLinVals - 32 ? src[32 + lane] : FP(0);
    }
#pragma unroll
    for (int u = 0; u < B; ++u)
      if (q0 + u < end) {
        a0 += v0[u];
        a1 += v1[u];
      }
  }
}

template <typename FP, typename SP>
__global__ void __launch_bounds__(32 * kCamWarps) k_lin_cams(Dev<FP, SP> d, int force, int phase) {
  if (!force && !d.st->do_linearize) return;
  __shared__ FP scratch[32];
  const int lane = threadIdx.x & 31;
  const uint32_t c = blockIdx.x * kCamWarps + (threadIdx.x >> 5);
  if (phase == 1) {
    if (c < d.nc) {
      FP a0 = FP(0), a1 = FP(0);
      lin_cam_sum(d, c, lane, a0, a1);
      d.red[54ull * c + lane] = a0;
      if (lane < kLinVals - 32) d.red[54ull * c + 32 + lane] = a1;
    }
    if (last_block(&d.st->cnt[0])) {
      const FP chi = reduce_partials(d.tile_red, d.ntiles, scratch);
      const FP m1 = reduce_partials_max(d.tile_red2, d.ntiles, scratch);
      int bad = 0;
      for (uint32_t i = threadIdx.x; i < d.ntiles; i += blockDim.x) bad += __ldcg(d.tile_flag + i) ? 0 : 1;
      bad = __syncthreads_count(bad > 0);
      if (threadIdx.x == 0) {
        d.red[red_scalars(d) + kRedLinChi] = chi;
        d.red[red_scalars(d) + kRedLinFail] = FP(bad);
        d.redmax[kRedMaxLin] = m1;
      }
    }
    return;
  }
  if (c < d.nc && d.jfact && lane == 0) {  // factored J store: R and f per camera
    // R as the edges used it (the camera's precomputed record), f
#pragma unroll
    for (int k = 0; k < 9; ++k) d.Rf[10ull * c + k] = d.cpre[static_cast<uint64_t>(kCamPre) * c + 8 + k];
    d.Rf[10ull * c + 9] = d.x[9ull * c + 6];
  }
  FP gm_t = FP(0);  // per thread: its warp's camera (uniform over the warp)
  int fin_t = 1;
  if (c < d.nc) {
    FP a0 = FP(0), a1 = FP(0);
    if (phase == 0) {
      lin_cam_sum(d, c, lane, a0, a1);
    } else {
      a0 = d.red[54ull * c + lane];
      if (lane < kLinVals - 32) a1 = d.red[54ull * c + 32 + lane];
    }
    const bool freev = d.col_free[9ull * c];
    // value v lives in lane v (a0) or lane v-32 (a1)
    if (lane < 9) d.b[9ull * c + lane] = freev ? a0 : FP(0);
    if (lane >= 9) d.Hc[45ull * c + (lane - 9)] = freev ? a0 : FP(0);
    if (lane < kLinVals - 32) d.Hc[45ull * c + (lane + 32 - 9)] = freev ? a1 : FP(0);
    // diagonal H(k,k) sits at value 9 + p9(k,k)
    const int k = lane < 9 ? lane : 0;
    const int v = 9 + p9(k, k);
    const FP from0 = __shfl_sync(0xffffffffu, a0, v & 31);
    const FP from1 = __shfl_sync(0xffffffffu, a1, v & 31);
    const FP diag = v < 32 ? from0 : from1;
    FP gm = FP(0);
    int fin = 1;
    if (lane < 9) {
      const FP cl = clampv(diag, FP(d.st->clamp_min), FP(d.st->clamp_max));
      d.clamped[9ull * c + lane] = freev ? cl : FP(0);
      d.D[9ull * c + lane] = freev ? FP(1) / sqrt(cl) : FP(0);
      if (freev) {
        fin = (is_finite(a0) && is_finite(diag)) ? 1 : 0;
        gm = fabs(a0);
      }
    }
    gm_t = gm;
    fin_t = fin;
  }
  // this block's cameras (max |b|, finiteness) and, when fused, its fixed slice
  // of the tiles' chi^2 / max |b| / flag partials: the last block then folds
  // one partial per block instead of every tile's (fixed order, deterministic)
  FP chi_t = FP(0);
  if (phase == 0) {
    const uint32_t per = (d.ntiles + gridDim.x - 1) / gridDim.x;
    const uint32_t lo = min(d.ntiles, per * blockIdx.x), hi = min(d.ntiles, lo + per);
    for (uint32_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
      chi_t += __ldcg(d.tile_red + i);
      gm_t = fmax(gm_t, __ldcg(d.tile_red2 + i));
      fin_t &= __ldcg(d.tile_flag + i) ? 1 : 0;
    }
  }
  const FP bchi = block_sum(chi_t, scratch);
  const FP bmax = block_max(gm_t, scratch);
  const int bfin = __syncthreads_and(fin_t);
  if (threadIdx.x == 0) {
    d.blk_red[blockIdx.x] = bchi;
    d.blk_red2[blockIdx.x] = bmax;
    d.blk_flag[blockIdx.x] = bfin;
  }
  if (last_block(&d.st->cnt[0])) {
    const FP m = reduce_partials_max(d.blk_red2, gridDim.x, scratch);
    const int f = reduce_flags_and(d.blk_flag, gridDim.x);
    if (phase == 0) {
      const FP chi = reduce_partials(d.blk_red, gridDim.x, scratch);
      if (threadIdx.x == 0) fin_lin(d.st, chi, f != 0, m);
    } else if (threadIdx.x == 0) {
      const FP* rs = d.red + red_scalars(d);
      fin_lin(d.st, rs[kRedLinChi], f != 0 && rs[kRedLinFail] == FP(0), fmax(d.redmax[kRedMaxLin], m));
    }
  }
}

// lambda0 = tau * max over free columns of D^2 * clamped (linear_system.hpp:94-99)
template <typename FP, typename SP>
__global__ void k_init_damping(Dev<FP, SP> d) {
  __shared__ FP scratch[32];
  FP m = FP(0);
  bool any = false;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < d.ncols;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    if (d.col_free[i] && counted(d, i)) {
      any = true;
      m = fmax(m, d.D[i] * d.D[i] * d.clamped[i]);
    }
  m = block_max(m, scratch);
  const int anyb = __syncthreads_or(any);
  if (threadIdx.x == 0) {
    d.blk_red[blockIdx.x] = m;
    d.blk_flag[blockIdx.x] = anyb;
  }
  if (last_block(&d.st->cnt[1])) {
    const FP mm = reduce_partials_max(d.blk_red, gridDim.x, scratch);
    const int a = reduce_flags_or(d.blk_flag, gridDim.x);
    if (threadIdx.x == 0) {
      if (!d.dist) {
        fin_damp(d.st, mm, a != 0);
      } else {
        d.redmax[kRedMaxDamp] = mm;
        d.red[red_scalars(d) + kRedDampAny] = FP(a ? 1 : 0);
      }
    }
  }
}

// =====================================================================
// LM iteration prologue (levenberg_marquardt.hpp:149-169): one thread.
// =====================================================================
template <typename FP>
__global__ void k_iter_begin(State<FP>* st, gb_iteration_record* recs) {
  if (st->terminated) {
    st->iter_active = 0;
    return;
  }
  const int it = ++st->lm_it;
  gb_iteration_record& rec = recs[it - 1];
  rec = gb_iteration_record{};
  rec.iteration = it;
  rec.chi2_before = static_cast<double>(st->chi2);
  rec.lambda = static_cast<double>(st->lambda);
  st->iter_active = 0;
  st->accepted = 0;
  st->do_linearize = 0;
  if (!st->lin_finite) {
    rec.chi2_after = rec.chi2_before;
    st->termination = GB_TERM_NON_FINITE_LINEARIZATION;
    st->terminated = 1;
    return;
  }
  if (st->grad_max < static_cast<FP>(st->grad_tol)) {
    rec.chi2_after = rec.chi2_before;
    st->termination = GB_TERM_GRADIENT_SMALL;
    st->terminated = 1;
    return;
  }
  st->iter_active = 1;
  st->lambda_solve = st->lambda;
  st->pcg_done = 0;
  st->pcg_it = 0;
  st->dir_pending = 0;
  st->x_pending = 0;
  st->pcg_conv = 0;
  st->pcg_zero = 0;
  st->pcg_relres = 0.0;
  st->fallbacks = 0;
}

// =====================================================================
// Block-Jacobi preconditioner (LinearSystem::build_preconditioner,
// linear_system.hpp:120-160): B = D H D + damp, lower Cholesky (LLT), inverse
// L^-T L^-1 stored packed; non-SPD or non-finite inverse -> clamped diagonal
// inverse fallback (counted). One thread per vertex (cameras, then points).
// =====================================================================
template <typename FP, int N>
__device__ inline bool chol_inverse(FP (&B)[N * (N + 1) / 2], FP* out_packed) {
  // B: packed upper row-major == packed lower column-major; L stored in place
  // as lower row-major packed: L(i,j) (j<=i) at i*(i+1)/2 + j.
  FP L[N * (N + 1) / 2];
  auto up = [](int i, int j) { return i * N - i * (i - 1) / 2 + (j - i); };  // i <= j
  auto lo = [](int i, int j) { return i * (i + 1) / 2 + j; };                // j <= i
#pragma unroll
  for (int k = 0; k < N; ++k) {
    FP x = B[up(k, k)];
#pragma unroll
    for (int j = 0; j < k; ++j) x -= L[lo(k, j)] * L[lo(k, j)];
    if (!(x > FP(0)) && !(x != x)) return false;  // Eigen fails on x <= 0; NaN propagates
    x = sqrt(x);
    L[lo(k, k)] = x;
#pragma unroll
    for (int i = k + 1; i < N; ++i) {
      FP v = B[up(k, i)];
#pragma unroll
      for (int j = 0; j < k; ++j) v -= L[lo(i, j)] * L[lo(k, j)];
      L[lo(i, k)] = v / x;
    }
  }
  // Linv (lower) in place: forward substitution on the identity
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const FP dii = FP(1) / L[lo(i, i)];
#pragma unroll
    for (int j = 0; j < i; ++j) {
      FP v = FP(0);
#pragma unroll
      for (int k = j; k < i; ++k) v -= L[lo(i, k)] * L[lo(k, j)];
      L[lo(i, j)] = v * dii;
    }
    L[lo(i, i)] = dii;
  }
  // inv = Linv^T Linv, upper packed
  bool ok = true;
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = i; j < N; ++j) {
      FP v = FP(0);
#pragma unroll
      for (int k = j; k < N; ++k) v += L[lo(k, i)] * L[lo(k, j)];
      out_packed[up(i, j)] = v;
      ok = ok && is_finite(v);
    }
  return ok;
}

template <typename FP, typename SP, int N>
__device__ inline void precond_vertex(const Dev<FP, SP>& d, const FP* H, FP* M, uint64_t col, bool freev) {
  constexpr int NP = N * (N + 1) / 2;
  if (!freev) {
#pragma unroll
    for (int k = 0; k < NP; ++k) M[k] = FP(0);
    return;
  }
  const FP lam = d.st->lambda_solve;
  FP Dv[N];
#pragma unroll
  for (int k = 0; k < N; ++k) Dv[k] = d.D[col + k];
  FP B[NP];
  int q = 0;
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = i; j < N; ++j, ++q) {
      B[q] = Dv[i] * H[q] * Dv[j];
      if (i == j) B[q] += d.st->before_scaling ? lam * Dv[i] * Dv[i] : lam;
    }
  FP out[NP];
  if (!chol_inverse<FP, N>(B, out)) {
    FP diag[N];
    q = 0;
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int j = i; j < N; ++j, ++q)
        if (i == j) diag[i] = clampv(B[q], FP(d.st->clamp_min), FP(d.st->clamp_max));
    q = 0;
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int j = i; j < N; ++j, ++q) out[q] = (i == j) ? FP(1) / diag[i] : FP(0);
    if (d.rank == 0 || N == 3) atomicAdd(&d.st->fallbacks, 1);  // replicated camera blocks counted once
  }
#pragma unroll
  for (int k = 0; k < NP; ++k) M[k] = out[k];
}

// Block-Jacobi build + inversion (linear_system.hpp:120-160). Cameras (9x9,
// register-heavy) and points (3x3) are separate kernels so the point pass
// runs at full occupancy.
template <typename FP, typename SP>
__global__ void k_precond_cams(Dev<FP, SP> d) {
  if (!d.st->iter_active || d.st->schur) return;  // Schur: k_schur_pre_cams
  for (uint64_t v = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; v < d.nc;
       v += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t col = 9 * v;
    precond_vertex<FP, SP, 9>(d, d.Hc + 45 * v, d.Mc + 45 * v, col, d.col_free[col]);
  }
}
template <typename FP, typename SP>
__global__ void __launch_bounds__(256) k_precond_pts(Dev<FP, SP> d) {
  if (!d.st->iter_active) return;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < d.np;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t col = 9ull * d.nc + 3 * i;
    precond_vertex<FP, SP, 3>(d, d.Hp + 6 * i, d.Mp + 6 * i, col, d.col_free[col]);
  }
}

// z = M r for one vertex (LinearSystem::apply_preconditioner,
// linear_system.hpp:164-180): FP accumulation, narrowed to SP.
template <typename FP, typename SP, int N>
__device__ inline void apply_block(const FP* M, const SP* r, SP* z, FP* rz, FP* rr) {
  FP rv[N];
#pragma unroll
  for (int k = 0; k < N; ++k) rv[k] = widen<FP>(r[k]);
#pragma unroll
  for (int i = 0; i < N; ++i) {
    FP acc = FP(0);
#pragma unroll
    for (int j = 0; j < N; ++j) acc += M[i <= j ? i * N - i * (i - 1) / 2 + (j - i) : j * N - j * (j - 1) / 2 + (i - j)] * rv[j];
    const SP zi = narrow<SP>(acc);
    z[i] = zi;
    *rz += rv[i] * widen<FP>(zi);
    *rr += rv[i] * rv[i];
  }
}

// z = M r for one N-column block from register values of r (already
// narrowed to SP and widened back, exactly what apply_block re-reads)
template <typename FP, typename SP, int N>
__device__ inline void apply_block_reg(const FP* M, const FP (&rv)[N], SP* z, FP* rz, FP* rr) {
#pragma unroll
  for (int i = 0; i < N; ++i) {
    FP acc = FP(0);
#pragma unroll
    for (int j = 0; j < N; ++j) acc += M[i <= j ? i * N - i * (i - 1) / 2 + (j - i) : j * N - j * (j - 1) / 2 + (i - j)] * rv[j];
    const SP zi = narrow<SP>(acc);
    z[i] = zi;
    *rz += rv[i] * widen<FP>(zi);
    *rr += rv[i] * rv[i];
  }
}

// =====================================================================
// PCG (pcg_solve, pcg.hpp:34-105) on (D H D + damp) with block Jacobi.
// =====================================================================

// rhs = -D b; ||rhs|| (pcg.hpp:303-310, linear_system.hpp:188-189)
template <typename FP, typename SP>
__global__ void k_rhs_norm(Dev<FP, SP> d) {
  if (!d.st->iter_active) return;
  __shared__ FP scratch[32];
  FP acc = FP(0);
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < d.ncols;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    if (d.st->schur && i >= 9ull * d.nc) break;
    const FP rhs = d.st->schur ? d.rc[i] : -d.D[i] * d.b[i];
    if (counted(d, i)) acc += rhs * rhs;
  }
  acc = block_sum(acc, scratch);
  if (threadIdx.x == 0) d.blk_red[blockIdx.x] = acc;
  if (last_block(&d.st->cnt[2])) {
    const FP s = reduce_partials(d.blk_red, gridDim.x, scratch);
    if (threadIdx.x == 0) {
      if (!d.dist) {
        fin_rhs(d.st, s);
      } else {
        d.red[red_scalars(d) + kRedRhs] = s;
        d.red[red_scalars(d) + kRedFallback] = FP(d.st->fallbacks);
      }
    }
  }
}

// r = narrow(rhs * scale), x = 0, z = M r, p = z, rho = r.z, res = |r|
// r = narrow(rhs * scale), x = 0, z = M r, p = z, vt = D p for one vertex block
template <typename FP, typename SP, int N>
__device__ inline void pcg_init_block(const Dev<FP, SP>& d, uint64_t col, const FP* M, FP scale, FP* rz, FP* rr) {
  using A = arith_t<SP>;
  FP Dv[N], rv[N];
#pragma unroll
  for (int k = 0; k < N; ++k) {
    Dv[k] = d.D[col + k];
    const FP rhs = d.st->schur ? d.rc[col + k] : -Dv[k] * d.b[col + k];
    const SP rn = narrow<SP>(rhs * scale);
    d.r[col + k] = rn;
    d.xs[col + k] = narrow<SP>(FP(0));
    rv[k] = widen<FP>(rn);
  }
  SP zs[N];
  apply_block_reg<FP, SP, N>(M, rv, zs, rz, rr);
#pragma unroll
  for (int k = 0; k < N; ++k) {
    d.z[col + k] = zs[k];
    d.p[col + k] = zs[k];
    d.vt[col + k] = static_cast<A>(Dv[k]) * widen<A>(zs[k]);
  }
}

template <typename FP, typename SP>
__global__ void k_pcg_init(Dev<FP, SP> d) {
  if (!d.st->iter_active) return;
  __shared__ FP scratch[32];
  const FP scale = d.st->scale;
  FP rz = FP(0), rr = FP(0);
  const uint64_t nv = d.st->schur ? static_cast<uint64_t>(d.nc) : static_cast<uint64_t>(d.nc) + d.np;
  for (uint64_t v = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; v < nv;
       v += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const bool cam = v < d.nc;
    const uint64_t col = cam ? 9 * v : 9ull * d.nc + 3 * (v - d.nc);
    FP lrz = FP(0), lrr = FP(0);
    if (cam)
      pcg_init_block<FP, SP, 9>(d, col, d.Mc + 45 * v, scale, &lrz, &lrr);
    else
      pcg_init_block<FP, SP, 3>(d, col, d.Mp + 6 * (v - d.nc), scale, &lrz, &lrr);
    if (counted(d, col)) {
      rz += lrz;
      rr += lrr;
    }
  }
  rz = block_sum(rz, scratch);
  rr = block_sum(rr, scratch);
  if (threadIdx.x == 0) {
    d.blk_red[blockIdx.x] = rz;
    d.blk_red2[blockIdx.x] = rr;
  }
  if (last_block(&d.st->cnt[3])) {
    const FP srz = reduce_partials(d.blk_red, gridDim.x, scratch);
    const FP srr = reduce_partials(d.blk_red2, gridDim.x, scratch);
    if (threadIdx.x == 0) {
      if (!d.dist) {
        fin_init(d.st, srz, srr);
      } else {
        d.red[red_scalars(d) + kRedInitRz] = srz;
        d.red[red_scalars(d) + kRedInitRr] = srr;
      }
    }
  }
}

// HVP, point side + camera runs (LinearSystem::hvp linear_system.hpp:104-115,
// hvp_forward factor_descriptor.hpp:372-407, hvp_scatter :409-433). One CTA
// per tile (<= 512 edges in 256-edge chunks; heavy single-point tiles are
// chunked with a running point sum). D*p is pre-gathered into vt by the kernel
// that produced p, so an edge needs its J row, two indices and two L1/L2
// gathers (its camera's 9 and its point's 3 values). Camera Jc^T q: warp-
// segmented runs -> partial slots. Point Jp^T q: staged in shared memory and
// summed per point in slot order after the single tile barrier. The tile's
// p.Ap goes out as one partial per warp (no block reduction).
template <typename FP, typename SP, bool DYN, int MINB = 1>
__global__ void __launch_bounds__(kTileThreads, MINB) k_hvp_tiles(Dev<FP, SP> d, const uint32_t* list) {
  using A = arith_t<SP>;
  if (!d.st->iter_active || d.st->pcg_done) return;
  __shared__ A stage[kTileEdges * 3];
  __shared__ A hacc[3];
  __shared__ FP sX[DYN ? kTilePoints * 3 : 1];
  __shared__ __align__(16) A gsh[9 * kGsStride];
  const int tid = threadIdx.x, lane = tid & 31;
  const uint64_t pcol0 = 9ull * d.nc;
  const uint32_t t = list ? list[blockIdx.x] : blockIdx.x;
  const uint32_t eb = d.tile_ebeg[t], ne_t = d.tile_ecnt[t];
  const uint32_t pb = d.tile_pbeg[t], npt = d.tile_pbeg[t + 1] - pb;
  const bool heavy = ne_t > static_cast<uint32_t>(kTileEdges);
  const A* vtp = d.vt + pcol0 + 3ull * pb;
  if (DYN) {
    for (uint32_t i = tid; i < npt * 3; i += blockDim.x) sX[i] = d.x[pcol0 + 3ull * pb + i];
  }
  if (heavy && tid < 3) hacc[tid] = A(0);
  if (DYN || heavy) __syncthreads();

  for (uint32_t c0 = 0; c0 < ne_t; c0 += kTileThreads) {
    const uint32_t j = c0 + tid;
    const bool valid = j < ne_t;
    const uint32_t e = eb + (valid ? j : 0);
    const uint32_t cam = d.d_cam[e];
    const uint32_t lp = d.d_lpt[e];
    A jc[18], jp[6];
    if (DYN) {
      FP cp[9], fjc[18], fjp[6];
#pragma unroll
      for (int k = 0; k < 9; ++k) cp[k] = d.x[9ull * cam + k];
      snavely_linearize<FP>(cp, &sX[3 * lp], FP(0), FP(0), nullptr, fjc, fjp, nullptr,
                            d.cpre + static_cast<uint64_t>(kCamPre) * cam);
#pragma unroll
      for (int k = 0; k < 18; ++k) jc[k] = static_cast<A>(fjc[k]);
#pragma unroll
      for (int k = 0; k < 6; ++k) jp[k] = static_cast<A>(fjp[k]);
    } else {
      load_J(d, e, cam, jc, jp);
    }
    const A wgt = d.w ? static_cast<A>(d.w[e]) : A(1);
    const A* cv = d.vt + 9ull * cam;
    const A* pv = vtp + 3 * lp;
    A u0 = A(0), u1 = A(0), s0 = A(0), s1 = A(0);
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      const A v = cv[k];
      u0 += jc[k] * v;
      u1 += jc[9 + k] * v;
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const A v = pv[k];
      s0 += jp[k] * v;
      s1 += jp[3 + k] * v;
    }
    u0 += s0;
    u1 += s1;
    const A q0 = valid ? wgt * u0 : A(0), q1 = valid ? wgt * u1 : A(0);
    A g[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) g[k] = jc[k] * q0 + jc[9 + k] * q1;
    const uint32_t chunk = d.tile_chunk_base[t] + (c0 + (tid & ~31)) / 32;
    {
      const uint32_t prev = __shfl_up_sync(0xffffffffu, cam, 1);
      const unsigned hm = __ballot_sync(0xffffffffu, valid && (lane == 0 || cam != prev));
      const unsigned vm = __ballot_sync(0xffffffffu, valid);
      camera_runs<A, FP>(g, lane, hm, vm, hm ? d.chunk_part_base[chunk] : 0u, gsh + (tid & ~31), kGsStride, d.part,
                         d.run_slot);
    }
    A h[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) h[k] = jp[k] * q0 + jp[3 + k] * q1;
    if (!heavy) {
      if (valid)
#pragma unroll
        for (int k = 0; k < 3; ++k) stage[j * 3 + k] = h[k];
    } else {
#pragma unroll
      for (int k = 0; k < 3; ++k) stage[tid * 3 + k] = valid ? h[k] : A(0);
      __syncthreads();
      if (tid < 3) {
        A acc = hacc[tid];
        const uint32_t nvalid = min(static_cast<uint32_t>(kTileThreads), ne_t - c0);
        for (uint32_t q = 0; q < nvalid; ++q) acc += stage[q * 3 + tid];
        hacc[tid] = acc;
      }
      __syncthreads();
    }
  }
  __syncthreads();

  const A lam = static_cast<A>(d.st->lambda_solve);
  const int before = d.st->before_scaling;
  FP dot = FP(0);
  for (uint32_t i = tid; i < npt; i += blockDim.x) {
    A acc[3];
    if (heavy) {
#pragma unroll
      for (int k = 0; k < 3; ++k) acc[k] = hacc[k];
    } else {
      acc[0] = acc[1] = acc[2] = A(0);
      for (uint32_t q = d.pt_slot_off[pb + i]; q < d.pt_slot_off[pb + i + 1]; ++q) {
        const uint32_t sl = d.pt_slots[q];
#pragma unroll
        for (int k = 0; k < 3; ++k) acc[k] += stage[sl * 3 + k];
      }
    }
    const uint64_t col = pcol0 + 3ull * (pb + i);
    const bool freev = d.col_free[col];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const FP Dk = d.D[col + k];
      const A damp = before ? static_cast<A>(static_cast<FP>(d.st->lambda_solve) * Dk * Dk) : lam;
      const SP pk = d.p[col + k];
      const A out = freev ? damp * widen<A>(pk) + static_cast<A>(Dk) * acc[k] : A(0);
      const SP o = narrow<SP>(out);
      d.ap[col + k] = o;
      if (d.dbg_out) d.dbg_out[col + k] = out;
      dot += widen<FP>(pk) * widen<FP>(o);
    }
  }
  dot = warp_sum(dot);
  if (lane == 0) d.tile_red[8ull * t + (tid >> 5)] = dot;
}

// vt = (Arith) D * widen(p) for every column (the HVP's gather source).
template <typename FP, typename SP>
__global__ void k_make_vt(Dev<FP, SP> d) {
  using A = arith_t<SP>;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < d.ncols;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    d.vt[i] = static_cast<A>(d.D[i]) * widen<A>(d.p[i]);
}

// =====================================================================
// Normal-tile kernels (<= kTileEdges edges, <= kTileCams cameras): one CTA
// pass per tile, one edge per thread. The tile's cameras are staged in shared
// memory by the prologue (the edge loop reads a 16-bit local camera index),
// so each edge costs one dependent DRAM round trip (its J row, indices).
// =====================================================================

// Linearize (factor_descriptor.hpp:272-292, :322-370, unscaled half of
// :435-482) on a normal tile. Camera b + packed H: every edge's Jc rows,
// w r and w are staged in shared memory; each warp then reduces its own
// 32-edge chunk run by run with one lane per output value (54 values over
// 32 lanes), i.e. plain FMAs over shared memory instead of shuffle trees.
// Dynamic shared memory: see lin_normal_smem().

// One edge's contribution to camera value V of its run: V < 9 is b_V = Jc0V w r0
// + Jc1V w r1, V in [9, 54) is H(i, j) = w (Jc0i Jc0j + Jc1i Jc1j) (packed upper).
template <typename FP, int V>
__device__ __forceinline__ FP lin_cam_value(const FP* jc, FP wr0, FP wr1, FP w) {
  if constexpr (V < 9) {
    return jc[V] * wr0 + jc[9 + V] * wr1;
  } else if constexpr (V >= kLinVals) {
    return FP(0);
  } else {
    constexpr int i = p9row(V - 9), k = p9col(V - 9);
    return w * (jc[i] * jc[k] + jc[9 + i] * jc[9 + k]);
  }
}

// first butterfly step (xor 16): values I and I + 32 generated in pairs
template <typename FP, int... I>
__device__ __forceinline__ void lin_shfl_first(FP* v, bool hi, const FP* jc, FP wr0, FP wr1, FP w,
                                               std::integer_sequence<int, I...>) {
  ((v[I] = [&] {
     const FP a = lin_cam_value<FP, I>(jc, wr0, wr1, w);
     const FP b = lin_cam_value<FP, I + 32>(jc, wr0, wr1, w);
     return (hi ? b : a) + __shfl_xor_sync(0xffffffffu, hi ? a : b, 16);
   }()),
   ...);
}

template <typename FP, int O>
__device__ __forceinline__ void lin_shfl_step(FP* v, int lane) {
  const bool hi = lane & O;
#pragma unroll
  for (int i = 0; i < 2 * O; ++i) {
    const FP keep = hi ? v[i + 2 * O] : v[i], send = hi ? v[i] : v[i + 2 * O];
    v[i] = keep + __shfl_xor_sync(0xffffffffu, send, O);
  }
}

// Sum of the 54 camera values over the lanes with `in` set, written to dst[0,
// 54). Lanes outside zero their inputs (so their values are exactly +0, even
// where a Jacobian entry is not finite); then a transposing butterfly (each xor step halves the values a lane holds,
// 62 fp64 shuffles per warp) instead of shared-memory staging; lane l ends
// with values 2l and 2l+1.
template <typename FP>
__device__ __forceinline__ void lin_cam_shfl(bool in, const FP* jc_in, FP wr0, FP wr1, FP w, int lane, FP* dst) {
  FP jc[18];
#pragma unroll
  for (int k = 0; k < 18; ++k) jc[k] = in ? jc_in[k] : FP(0);
  if (!in) wr0 = wr1 = w = FP(0);
  FP v[32];
  lin_shfl_first<FP>(v, (lane & 16) != 0, jc, wr0, wr1, w, std::make_integer_sequence<int, 32>{});
  lin_shfl_step<FP, 8>(v, lane);
  lin_shfl_step<FP, 4>(v, lane);
  lin_shfl_step<FP, 2>(v, lane);
  lin_shfl_step<FP, 1>(v, lane);
  if (2 * lane < kLinVals) {
    dst[2 * lane] = v[0];
    dst[2 * lane + 1] = v[1];
  }
}

// 128-thread CTAs (four passes over a 512-edge tile), four per SM: while one
// CTA waits at a barrier or on its prologue gathers, three others compute.
// tile record, one per normal tile (list order)
// kMSlot0 / kMNruns: the tile's camera-run slots [slot0, slot0 + nruns) (filled on the device by k_tile_aux)
enum TileMeta : int { kMT = 0, kMEb, kMNe, kMPb, kMNpt, kMCb, kMNcam, kMCh0, kMAux16, kMLin16, kMSlot0, kMNruns, kMCount };

// Recompute-HVP per-tile lin blob (hvp_rc.cuh): written per linearization by
// k_lin_normal (recompute path) or k_tile_lin_rc.
constexpr int kRcRec = 16;   // per-camera record stride (static [R t f k1 k2 0], dynamic [M v_t v_int 0])
__host__ __device__ constexpr uint32_t rc_r16(uint64_t b) { return static_cast<uint32_t>((b + 15) / 16 * 16); }
// lin blob of the recompute path (per linearization): point D, tile camera
// static records, Huber weights, point parameters X
struct RcLinSec {
  uint32_t D, cam, w, X, bytes;
};
template <typename FP>
__host__ __device__ inline RcLinSec rc_lin_sections(uint32_t ne, uint32_t npt, uint32_t ncam, bool huber) {
  const uint32_t ne8 = (ne + kEdgePad - 1) / kEdgePad * kEdgePad;
  RcLinSec l;
  l.D = 0;
  l.cam = l.D + rc_r16(sizeof(FP) * 3ull * npt);
  l.w = l.cam + rc_r16(sizeof(FP) * static_cast<uint64_t>(kRcRec) * ncam);
  l.X = l.w + (huber ? rc_r16(sizeof(FP) * 1ull * ne8) : 0u);
  l.bytes = l.X + rc_r16(sizeof(FP) * 3ull * npt);
  return l;
}


constexpr int kLinThreads = 128;
template <typename FP>
__host__ __device__ constexpr size_t lin_normal_smem() {
  return sizeof(FP) * (kTilePoints * 3 + kTileCams * 9 + kTileEdges * 9 + 32 + kTileCams * kCamPre);
}

template <typename FP, typename SP, bool STORE, bool AUTO>
__global__ void __launch_bounds__(kLinThreads, 4) k_lin_normal(Dev<FP, SP> d, int force) {
  if (!force && !d.st->do_linearize) return;
  extern __shared__ __align__(16) unsigned char lin_smem[];
  FP* sX = reinterpret_cast<FP*>(lin_smem);
  FP* sC = sX + kTilePoints * 3;
  FP* pst = sC + kTileCams * 9;
  FP* scratch = pst + kTileEdges * 9;
  FP* sPre = scratch + 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t t = d.normal_tiles[blockIdx.x];
  const uint32_t eb = d.tile_ebeg[t], ne_t = d.tile_ecnt[t];
  const uint32_t pb = d.tile_pbeg[t], npt = d.tile_pbeg[t + 1] - pb;
  const uint32_t cb = d.tile_cam_off[t], ncam = d.tile_cam_off[t + 1] - cb;
  const uint64_t pcol0 = 9ull * d.nc;
  for (uint32_t i = tid; i < npt * 3; i += blockDim.x) sX[i] = d.x[pcol0 + 3ull * pb + i];
  for (uint32_t i = tid; i < ncam * 9; i += blockDim.x) sC[i] = d.x[9ull * d.tile_cams[cb + i / 9] + i % 9];
  if (!AUTO)
    for (uint32_t i = tid; i < ncam * kCamPre; i += blockDim.x)
      sPre[i] = d.cpre[static_cast<uint64_t>(kCamPre) * d.tile_cams[cb + i / kCamPre] + i % kCamPre];
  // recompute path: this pass also writes the tile's per-linearization blob
  // (point D, camera records [R t f k1 k2], Huber w, point X; hvp_rc.cuh)
  const bool blob = !AUTO && d.part15 != nullptr;
  unsigned char* lb = blob ? d.tile_lin + 16ull * d.tile_meta[static_cast<uint64_t>(kMCount) * blockIdx.x + kMLin16]
                           : nullptr;
  const RcLinSec lsec = rc_lin_sections<FP>(ne_t, npt, ncam, d.w != nullptr);
  __syncthreads();
  if (blob) {
    FP* bx = reinterpret_cast<FP*>(lb + lsec.X);
    for (uint32_t i = tid; i < npt * 3; i += blockDim.x) bx[i] = sX[i];
    FP* bc = reinterpret_cast<FP*>(lb + lsec.cam);
    for (uint32_t k = tid; k < kRcRec * ncam; k += blockDim.x) {
      const uint32_t lc = k / kRcRec, v = k % kRcRec;
      bc[k] = v < 9 ? sPre[kCamPre * lc + 8 + v] : (v < 15 ? sC[9 * lc + v - 6] : FP(0));
    }
  }
  FP chi = FP(0);
  for (uint32_t c0 = 0; c0 < ne_t; c0 += kLinThreads) {
  const uint32_t j = c0 + tid;
  const bool valid = j < ne_t;
  const uint32_t e = eb + (valid ? j : 0);
  const uint32_t lc = d.d_lcam[e], lp = d.d_lpt[e];
  const FP o0 = d.d_obs[e], o1 = d.d_obs[static_cast<uint64_t>(d.na) + e];

  FP res[2], jc[18], jp[6], fac[10];
  if (AUTO) {
    snavely_residual<FP>(&sC[9 * lc], &sX[3 * lp], o0, o1, res);
    snavely_jacobians_auto<FP>(&sC[9 * lc], &sX[3 * lp], jc, jp);
  } else {
    snavely_linearize<FP>(&sC[9 * lc], &sX[3 * lp], o0, o1, res, jc, jp, fac, &sPre[kCamPre * lc]);
  }
  const FP s = res[0] * res[0] + res[1] * res[1];
  const FP w = valid ? loss_weight<FP>(d.loss_kind, d.huber, s) : FP(0);
  if (valid) chi += loss_value<FP>(d.loss_kind, d.huber, s);
  if (STORE) {
    if (valid) store_J(d, e, jc, jp, fac);
#pragma unroll
    for (int k = 0; k < 18; ++k) jc[k] = widen<FP>(narrow<SP>(jc[k]));
#pragma unroll
    for (int k = 0; k < 6; ++k) jp[k] = widen<FP>(narrow<SP>(jp[k]));
  }
  if (d.w && valid) {
    d.w[e] = w;
    if (blob) reinterpret_cast<FP*>(lb + lsec.w)[j] = w;
  }
  const FP wr0 = valid ? w * res[0] : FP(0), wr1 = valid ? w * res[1] : FP(0);
  if (valid) {
    FP* pv = pst + j * 9;
    pv[0] = jp[0] * wr0 + jp[3] * wr1;
    pv[1] = jp[1] * wr0 + jp[4] * wr1;
    pv[2] = jp[2] * wr0 + jp[5] * wr1;
    pv[3] = w * (jp[0] * jp[0] + jp[3] * jp[3]);
    pv[4] = w * (jp[0] * jp[1] + jp[3] * jp[4]);
    pv[5] = w * (jp[0] * jp[2] + jp[3] * jp[5]);
    pv[6] = w * (jp[1] * jp[1] + jp[4] * jp[4]);
    pv[7] = w * (jp[1] * jp[2] + jp[4] * jp[5]);
    pv[8] = w * (jp[2] * jp[2] + jp[5] * jp[5]);
  }
  // run structure of this warp's 32-edge chunk
  const unsigned full = 0xffffffffu;
  const uint32_t prev = __shfl_up_sync(full, lc, 1);
  const unsigned hm = __ballot_sync(full, valid && (lane == 0 || lc != prev));
  const unsigned vm = __ballot_sync(full, valid);
  const uint32_t slot0 = hm ? d.chunk_part_base[d.tile_chunk_base[t] + c0 / 32 + warp] : 0u;
  {
    // one register butterfly per camera run of the chunk (a tile's edges are
    // camera-sorted, so a chunk has ~1.5 runs on average)
    unsigned heads = hm;
    uint32_t run = 0;
    while (heads) {
      const int start = __ffs(heads) - 1;
      heads &= heads - 1;
      const int stop = heads ? __ffs(heads) - 1 : 32 - __clz(vm);
      lin_cam_shfl<FP>(lane >= start && lane < stop, jc, wr0, wr1, w, lane,
                       d.part + static_cast<uint64_t>(d.run_slot[slot0 + run]) * kLinVals);
      ++run;
    }
  }
  }
  __syncthreads();  // pst complete

  // point epilogue (same as the generic kernel)
  FP gmax = FP(0);
  int fin = 1;
  for (uint32_t i = tid; i < npt; i += blockDim.x) {
    FP acc[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) acc[k] = FP(0);
    for (uint32_t q = d.pt_slot_off[pb + i]; q < d.pt_slot_off[pb + i + 1]; ++q) {
      const uint32_t sl = d.pt_slots[q];
#pragma unroll
      for (int k = 0; k < 9; ++k) acc[k] += pst[sl * 9 + k];
    }
    const uint64_t col = pcol0 + 3ull * (pb + i);
    const bool freev = d.col_free[col];
    const uint64_t pidx = static_cast<uint64_t>(pb + i);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const FP bk = freev ? acc[k] : FP(0);
      d.b[col + k] = bk;
      const FP diag = freev ? acc[3 + p3(k, k)] : FP(0);
      const FP cl = clampv(diag, FP(d.st->clamp_min), FP(d.st->clamp_max));
      d.clamped[col + k] = freev ? cl : FP(0);
      const FP Dv = freev ? FP(1) / sqrt(cl) : FP(0);
      d.D[col + k] = Dv;
      if (blob) reinterpret_cast<FP*>(lb + lsec.D)[3 * i + k] = Dv;
      if (freev) {
        fin &= (is_finite(bk) && is_finite(diag)) ? 1 : 0;
        gmax = fmax(gmax, fabs(bk));
      }
    }
#pragma unroll
    for (int k = 0; k < 6; ++k) d.Hp[6 * pidx + k] = freev ? acc[3 + k] : FP(0);
  }
  const FP tchi = block_sum(chi, scratch);
  const FP tmax = block_max(gmax, scratch);
  const int tfin = __syncthreads_and(fin);
  if (tid == 0) {
    d.tile_red[t] = tchi;
    d.tile_red2[t] = tmax;
    d.tile_flag[t] = tfin;
  }
}

// Camera side of the HVP + p.Ap finalization (pcg.hpp:332-340). Each block
// also folds a fixed slice of the tiles' per-warp dot partials, so the last
// block only sums one partial per block (fixed order, deterministic).
// phase 0: fused (world == 1). phase 1: per-rank camera J^T q sums -> red[0,
// 9nc) and the local point dot -> red[9nc]. phase 2: ap_c from the allreduced
// sums, camera dot, pAp = camera dot + reduced point dot.
template <typename FP, typename SP>
__global__ void __launch_bounds__(32 * kCamWarps) k_hvp_cams(Dev<FP, SP> d, int phase) {
  using A = arith_t<SP>;
  if (!d.st->iter_active || d.st->pcg_done) return;
  __shared__ FP scratch[32];
  const int lane = threadIdx.x & 31;
  const uint32_t c = blockIdx.x * kCamWarps + (threadIdx.x >> 5);
  FP mine = FP(0);
  if (c < d.nc) {
    FP acc[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) acc[k] = FP(0);
    if (phase != 2) {
      for (uint32_t q = d.cam_part_off[c] + lane; q < d.cam_part_off[c + 1]; q += 32) {
        const FP* src = d.part + static_cast<uint64_t>(q) * 9;  // camera-major storage
#pragma unroll
        for (int k = 0; k < 9; ++k) acc[k] += src[k];
      }
#pragma unroll
      for (int k = 0; k < 9; ++k) acc[k] = warp_sum(acc[k]);
    }
    if (phase == 1) {
      if (lane < 9) {
        FP a = acc[0];
#pragma unroll
        for (int k = 1; k < 9; ++k)
          if (lane == k) a = acc[k];
        d.red[9ull * c + lane] = a;
      }
    } else {
      FP dot = FP(0);
      const bool freev = d.col_free[9ull * c];
      if (lane < 9) {
        const uint64_t col = 9ull * c + lane;
        FP a = acc[0];
#pragma unroll
        for (int k = 1; k < 9; ++k)
          if (lane == k) a = acc[k];
        if (phase == 2) a = d.red[col];
        const FP Dk = d.D[col];
        const A damp = d.st->before_scaling ? static_cast<A>(d.st->lambda_solve * Dk * Dk)
                                            : static_cast<A>(d.st->lambda_solve);
        const SP pk = d.p[col];
        const A out = freev ? damp * widen<A>(pk) + static_cast<A>(Dk) * static_cast<A>(a) : A(0);
        const SP o = narrow<SP>(out);
        d.ap[col] = o;
        if (d.dbg_out) d.dbg_out[col] = out;
        dot = widen<FP>(pk) * widen<FP>(o);
      }
      dot = warp_sum(dot);
      if (lane == 0) mine = dot;
    }
  }
  if (phase != 2) {  // this block's slice of the tiles' point dot partials
    const uint64_t ntp = 8ull * d.ntiles;
    const uint64_t per = (ntp + gridDim.x - 1) / gridDim.x;
    const uint64_t lo = min(ntp, per * blockIdx.x), hi = min(ntp, lo + per);
    for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) mine += d.tile_red[i];
  }
  const FP bsum = block_sum(mine, scratch);
  if (threadIdx.x == 0) d.blk_red[blockIdx.x] = bsum;
  if (last_block(&d.st->cnt[4])) {
    const FP tot = reduce_partials(d.blk_red, gridDim.x, scratch);
    if (threadIdx.x == 0) {
      if (phase == 0) fin_hvp(d.st, tot);
      else if (phase == 1) d.red[9ull * d.nc] = tot;
      else fin_hvp(d.st, tot + d.red[9ull * d.nc]);
    }
  }
}

// Finalize kernels for world > 1 (one thread; inputs already allreduced).
template <typename FP, typename SP>
__global__ void k_fin(Dev<FP, SP> d, int site) {
  State<FP>* st = d.st;
  const FP* rs = d.red + red_scalars(d);
  switch (site) {
    case 0:  // init damping
      fin_damp(st, d.redmax[kRedMaxDamp], rs[kRedDampAny] > FP(0));
      break;
    case 1:  // rhs norm + fallback count
      if (!st->iter_active) return;
      st->fallbacks = static_cast<int>(rs[kRedFallback]);
      fin_rhs(st, rs[kRedRhs]);
      break;
    case 2:  // pcg init
      if (!st->iter_active) return;
      fin_init(st, rs[kRedInitRz], rs[kRedInitRr]);
      break;
    case 3:  // pcg update
      if (!st->iter_active || st->pcg_done) return;
      fin_upd(st, rs[kRedUpdRz], rs[kRedUpdRr]);
      break;
    case 4:  // step
      if (!st->iter_active) return;
      fin_step(st, rs[kRedStepPred], rs[kRedStepFail] == FP(0));
      break;
    case 5:  // candidate chi^2
      if (!st->iter_active || !st->step_finite) return;
      st->chi2_new = rs[kRedChi];
      break;
  }
}

// x += alpha p; r -= alpha Ap; z = M r for one N-column vertex block, all
// loads issued before any store (the vectors are distinct arrays)
template <typename FP, typename SP>
__device__ inline SP pcg_x_value(SP x, SP p, FP alpha) {  // x += alpha p (pcg.hpp:340-357)
  return narrow<SP>(widen<FP>(x) + alpha * widen<FP>(p));
}

template <typename FP, typename SP, int N>
__device__ inline void pcg_update_block(const Dev<FP, SP>& d, uint64_t col, const FP* M, FP alpha, FP* rz, FP* rr) {
  SP xs[N], pv[N], rs[N], aps[N];
#pragma unroll
  for (int k = 0; k < N; ++k) {
    if (!d.defer_x) {
      xs[k] = d.xs[col + k];
      pv[k] = d.p[col + k];
    }
    rs[k] = d.r[col + k];
    aps[k] = d.ap[col + k];
  }
  FP rv[N];
#pragma unroll
  for (int k = 0; k < N; ++k) {
    if (!d.defer_x) d.xs[col + k] = pcg_x_value<FP, SP>(xs[k], pv[k], alpha);
    const SP rn = narrow<SP>(widen<FP>(rs[k]) - alpha * widen<FP>(aps[k]));
    d.r[col + k] = rn;
    rv[k] = widen<FP>(rn);
  }
  apply_block_reg<FP, SP, N>(M, rv, d.z + col, rz, rr);
}

template <typename FP, typename SP>
__device__ inline void pcg_update_vertex(const Dev<FP, SP>& d, uint64_t v, FP alpha, FP* rz, FP* rr) {
  const bool cam = v < d.nc;
  const uint64_t col = cam ? 9 * v : 9ull * d.nc + 3 * (v - d.nc);
  FP lrz = FP(0), lrr = FP(0);
  if (cam)
    pcg_update_block<FP, SP, 9>(d, col, d.Mc + 45 * v, alpha, &lrz, &lrr);
  else
    pcg_update_block<FP, SP, 3>(d, col, d.Mp + 6 * (v - d.nc), alpha, &lrz, &lrr);
  if (counted(d, col)) {
    *rz += lrz;
    *rr += lrr;
  }
}

// Two consecutive points per thread with 16-byte vector accesses (8-byte
// storage, 16-byte aligned point section): the same arithmetic per point as
// pcg_update_block<3>, a quarter of the memory instructions.
template <typename FP, typename SP>
__device__ inline void pcg_update_pair(const Dev<FP, SP>& d, uint64_t q, FP alpha, FP* rz, FP* rr) {
  static_assert(sizeof(SP) == 8 && sizeof(FP) == 8, "8-byte storage");
  const uint64_t col = 9ull * d.nc + 6 * q;
  double2 rv2[3], av2[3], xv2[3], pv2[3], mv2[6];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    rv2[k] = reinterpret_cast<const double2*>(d.r + col)[k];
    av2[k] = reinterpret_cast<const double2*>(d.ap + col)[k];
    if (!d.defer_x) {
      xv2[k] = reinterpret_cast<const double2*>(d.xs + col)[k];
      pv2[k] = reinterpret_cast<const double2*>(d.p + col)[k];
    }
  }
#pragma unroll
  for (int k = 0; k < 6; ++k) mv2[k] = reinterpret_cast<const double2*>(d.Mp + 12 * q)[k];
  const SP* rs = reinterpret_cast<const SP*>(rv2);
  const SP* as = reinterpret_cast<const SP*>(av2);
  const SP* xs = reinterpret_cast<const SP*>(xv2);
  const SP* ps = reinterpret_cast<const SP*>(pv2);
  const FP* M = reinterpret_cast<const FP*>(mv2);
  double2 ro2[3], zo2[3], xo2[3];
  SP* ro = reinterpret_cast<SP*>(ro2);
  SP* zo = reinterpret_cast<SP*>(zo2);
  SP* xo = reinterpret_cast<SP*>(xo2);
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    FP rvv[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const int i = 3 * j + k;
      if (!d.defer_x) xo[i] = pcg_x_value<FP, SP>(xs[i], ps[i], alpha);
      const SP rn = narrow<SP>(widen<FP>(rs[i]) - alpha * widen<FP>(as[i]));
      ro[i] = rn;
      rvv[k] = widen<FP>(rn);
    }
    FP lrz = FP(0), lrr = FP(0);
    apply_block_reg<FP, SP, 3>(M + 6 * j, rvv, zo + 3 * j, &lrz, &lrr);
    *rz += lrz;
    *rr += lrr;
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    reinterpret_cast<double2*>(d.r + col)[k] = ro2[k];
    reinterpret_cast<double2*>(d.z + col)[k] = zo2[k];
    if (!d.defer_x) reinterpret_cast<double2*>(d.xs + col)[k] = xo2[k];
  }
}

// x += alpha p; r -= alpha Ap; z = M r; rr, rz (pcg.hpp:340-357)
template <typename FP, typename SP>
__global__ void __launch_bounds__(256, sizeof(SP) == 8 ? 4 : 1) k_pcg_update(Dev<FP, SP> d) {
  if (!d.st->iter_active || d.st->pcg_done) return;
  __shared__ FP scratch[32];
  const FP alpha = d.st->alpha;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    d.st->dir_pending = 0;  // the HVP that consumed it has run
    if (d.defer_x) d.st->x_pending = 1;  // this update's x += alpha p goes to the next HVP (or k_step)
  }
  FP rz = FP(0), rr = FP(0);
  const uint64_t nv = d.st->schur ? static_cast<uint64_t>(d.nc) : static_cast<uint64_t>(d.nc) + d.np;
  const uint64_t gt = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  bool pairs = false;
  if constexpr (sizeof(SP) == 8 && sizeof(FP) == 8) pairs = !d.st->schur && (d.nc % 2) == 0;
  if (pairs) {  // cameras one per thread, then point pairs (an odd last point alone)
    for (uint64_t v = gt; v < d.nc; v += stride) pcg_update_vertex(d, v, alpha, &rz, &rr);
    if constexpr (sizeof(SP) == 8 && sizeof(FP) == 8)
      for (uint64_t q = gt; q < d.np / 2; q += stride) pcg_update_pair(d, q, alpha, &rz, &rr);
    if ((d.np & 1) && gt == 0) pcg_update_vertex(d, d.nc + d.np - 1, alpha, &rz, &rr);
  } else {
    for (uint64_t v = gt; v < nv; v += stride) pcg_update_vertex(d, v, alpha, &rz, &rr);
  }
  rz = block_sum(rz, scratch);
  rr = block_sum(rr, scratch);
  if (threadIdx.x == 0) {
    d.blk_red[blockIdx.x] = rz;
    d.blk_red2[blockIdx.x] = rr;
  }
  if (last_block(&d.st->cnt[5])) {
    const FP srz = reduce_partials(d.blk_red, gridDim.x, scratch);
    const FP srr = reduce_partials(d.blk_red2, gridDim.x, scratch);
    if (threadIdx.x == 0) {
      if (!d.dist) {
        fin_upd(d.st, srz, srr);
      } else {
        d.red[red_scalars(d) + kRedUpdRz] = srz;
        d.red[red_scalars(d) + kRedUpdRr] = srr;
      }
    }
  }
}

// p = narrow(z + beta p) (pcg.hpp:358-361), explicitly rounded so every
// kernel that applies it (k_pcg_dir, k_pcg_dir_rest, k_hvp_pipe) agrees bitwise
template <typename FP, typename SP>
__device__ inline SP pcg_dir_value(SP z, SP p, FP beta) {
  return narrow<SP>(fma_rn(beta, widen<FP>(p), widen<FP>(z)));
}

// Fused PCG step for the single-GPU path (cooperative launch): update
// (pcg.hpp:340-357), grid barrier, every block reduces the same partials in
// the same order (so beta and the stop decision agree everywhere), then
// p = z + beta p and vt = D p (pcg.hpp:358-361). Block 0 writes the state.
template <typename FP, typename SP>
__global__ void __launch_bounds__(256) k_pcg_step(Dev<FP, SP> d) {
  using A = arith_t<SP>;
  State<FP>* st = d.st;
  if (!st->iter_active || st->pcg_done) return;
  __shared__ FP scratch[32];
  const FP alpha = st->alpha, rho = st->rho, ref = st->ref_norm;
  const FP tol = static_cast<FP>(st->pcg_tol);
  const bool schur = st->schur;
  FP rz = FP(0), rr = FP(0);
  const uint64_t nv = schur ? static_cast<uint64_t>(d.nc) : static_cast<uint64_t>(d.nc) + d.np;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t v = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; v < nv; v += stride)
    pcg_update_vertex(d, v, alpha, &rz, &rr);
  rz = block_sum(rz, scratch);
  rr = block_sum(rr, scratch);
  if (threadIdx.x == 0) {
    d.blk_red[blockIdx.x] = rz;
    d.blk_red2[blockIdx.x] = rr;
  }
  cooperative_groups::this_grid().sync();
  const FP srz = reduce_partials(d.blk_red, gridDim.x, scratch);
  const FP srr = reduce_partials(d.blk_red2, gridDim.x, scratch);
  const FP res = sqrt(srr);
  const double rel = static_cast<double>(res / ref);
  const bool stop = !isfinite(rel) || res <= tol * ref;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->pcg_it += 1;
    st->pcg_relres = rel;
    if (!isfinite(rel)) {
      st->pcg_done = 1;
      st->pcg_conv = 0;
    } else if (res <= tol * ref) {
      st->pcg_done = 1;
      st->pcg_conv = 1;
    } else {
      st->beta = srz / rho;
      st->rho = srz;
    }
  }
  if (stop) return;
  const FP beta = srz / rho;
  const uint64_t n = schur ? 9ull * d.nc : d.ncols;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n; i += stride) {
    const SP pi = pcg_dir_value<FP, SP>(d.z[i], d.p[i], beta);
    d.p[i] = pi;
    d.vt[i] = static_cast<A>(d.D[i]) * widen<A>(pi);
  }
}

template <typename FP, typename SP>
__global__ void k_pcg_dir(Dev<FP, SP> d) {
  if (!d.st->iter_active || d.st->pcg_done) return;
  using A = arith_t<SP>;
  const FP beta = d.st->beta;
  const uint64_t n = d.st->schur ? 9ull * d.nc : d.ncols;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const SP pi = pcg_dir_value<FP, SP>(d.z[i], d.p[i], beta);
    d.p[i] = pi;
    d.vt[i] = static_cast<A>(d.D[i]) * widen<A>(pi);
  }
}

// k_pcg_dir for the columns the pipelined HVP does not update itself
// (hvp_pipe.cuh applies p = z + beta p to normal-tile points on the fly):
// cameras, with their per-tile copies tcv (cam_tc CSR), and the points of
// heavy tiles (column ranges). Arms dir_pending for k_hvp_pipe.
template <typename FP, typename SP>
__global__ void k_pcg_dir_rest(Dev<FP, SP> d, const uint64_t* rbeg, const uint64_t* rend, int nranges) {
  if (!d.st->iter_active || d.st->pcg_done) return;
  using A = arith_t<SP>;
  const FP beta = d.st->beta;
  if (blockIdx.x == 0 && threadIdx.x == 0) d.st->dir_pending = 1;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const uint64_t t0 = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  for (uint64_t i = t0; i < 9ull * d.nc; i += stride) {
    const SP pi = pcg_dir_value<FP, SP>(d.z[i], d.p[i], beta);
    d.p[i] = pi;
    const A v = static_cast<A>(d.D[i]) * widen<A>(pi);
    d.vt[i] = v;
    const uint64_t c = i / 9, k = i % 9;
    constexpr uint64_t CS = sizeof(A) == 8 ? 10 : 12;  // hvp_pipe.cuh cam_stride
    const uint32_t q1 = d.cam_tc_off[c + 1];
    for (uint32_t q = d.cam_tc_off[c]; q < q1; q += 8) {  // the camera's tile copies, 8 index loads in flight
      uint32_t tc[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) tc[u] = q + u < q1 ? d.cam_tc_idx[q + u] : 0u;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (q + u < q1) d.tcv[CS * tc[u] + k] = v;
    }
  }
  for (int r = 0; r < nranges; ++r)
    for (uint64_t i = rbeg[r] + t0; i < rend[r]; i += stride) {
      const SP pi = pcg_dir_value<FP, SP>(d.z[i], d.p[i], beta);
      d.p[i] = pi;
      d.vt[i] = static_cast<A>(d.D[i]) * widen<A>(pi);
    }
}

// Unscale, predicted decrease, dx = D x, candidate x_new = x + dx
// (pcg.hpp:364-365, linear_system.hpp:195-206, graph.hpp:126-128).
template <typename FP, typename SP>
__global__ void k_step(Dev<FP, SP> d) {
  if (!d.st->iter_active) return;
  __shared__ FP scratch[32];
  const FP unscale = d.st->unscale;
  const FP lam = d.st->lambda_solve;
  const int before = d.st->before_scaling;
  const bool zero = d.st->pcg_zero;
  const bool xpend = d.st->x_pending != 0;  // the last PCG update's deferred x += alpha p
  const FP alpha = d.st->alpha;
  FP pred = FP(0);
  int fin = 1;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < d.ncols;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    // every load before the first store (the compiler cannot reorder them
    // across the xs store, which would serialize two round trips per column)
    const FP Di = d.D[i];
    const bool ptcol = i >= 9ull * d.nc;
    const bool schur_pt = d.st->schur && ptcol;
    const SP xs0 = d.xs[i];
    const SP pv = xpend ? d.p[i] : xs0;
    const FP xpv = schur_pt ? d.xp[i - 9ull * d.nc] : FP(0);
    const FP bi = d.b[i];
    const FP xi = d.x[i];
    const bool fr = d.col_free[i];
    const SP xsn = xpend ? pcg_x_value<FP, SP>(xs0, pv, alpha) : xs0;
    if (xpend) d.xs[i] = xsn;
    const FP xsi = schur_pt ? xpv : (zero ? FP(0) : widen<FP>(xsn) * unscale);
    const FP rhs = -Di * bi;
    const FP damp = before ? lam * Di * Di : lam;
    if (counted(d, i)) pred += xsi * (damp * xsi + rhs);
    const FP dxi = Di * xsi;
    if (d.want_dx) d.dx[i] = dxi;
    if (!is_finite(dxi)) fin = 0;
    d.x_new[i] = fr ? xi + dxi : xi;
  }
  pred = block_sum(pred, scratch);
  fin = __syncthreads_and(fin);
  if (threadIdx.x == 0) {
    d.blk_red[blockIdx.x] = pred;
    d.blk_flag[blockIdx.x] = fin;
  }
  if (last_block(&d.st->cnt[6])) {
    const FP s = reduce_partials(d.blk_red, gridDim.x, scratch);
    const int f = reduce_flags_and(d.blk_flag, gridDim.x);
    if (threadIdx.x == 0) {
      d.st->x_pending = 0;
      if (!d.dist) {
        fin_step(d.st, s, f != 0);
      } else {
        d.red[red_scalars(d) + kRedStepPred] = s;
        d.red[red_scalars(d) + kRedStepFail] = f ? FP(0) : FP(1);
      }
    }
  }
}

// Candidate chi^2 at x_new (Graph::total_error_active graph.hpp:107-111,
// FactorDescriptor::evaluate_chi2 factor_descriptor.hpp:294-305); RAW=true
// gives raw_residual_sqnorm (:307-320) for BalGraph::mse. params: x or x_new.
template <typename FP, typename SP, bool RAW>
__global__ void __launch_bounds__(kTileThreads) k_chi2_tiles(Dev<FP, SP> d, const FP* params, int force) {
  if (!force && (!d.st->iter_active || !d.st->step_finite)) return;
  __shared__ FP scratch[32];
  const uint64_t pcol0 = 9ull * d.nc;
  // grid-stride over tiles (a fixed tile set and order per block), one
  // partial per block, so the last block folds gridDim.x values, not ntiles
  FP chi = FP(0);
  for (uint32_t t = blockIdx.x; t < d.ntiles; t += gridDim.x) {
    const uint32_t eb = d.tile_ebeg[t], ee = eb + d.tile_ecnt[t], pb = d.tile_pbeg[t];
    for (uint32_t e = eb + threadIdx.x; e < ee; e += blockDim.x) {
      const uint32_t cam = d.d_cam[e];
      FP cp[9];
#pragma unroll
      for (int k = 0; k < 9; ++k) cp[k] = params[9ull * cam + k];
      const FP* X = params + pcol0 + 3ull * (pb + d.d_lpt[e]);
      FP res[2];
      snavely_residual_pre<FP>(cp, d.cpre_new + static_cast<uint64_t>(kCamPre) * cam, X, d.d_obs[e],
                               d.d_obs[static_cast<uint64_t>(d.na) + e], res);
      const FP s = res[0] * res[0] + res[1] * res[1];
      chi += RAW ? s : loss_value<FP>(d.loss_kind, d.huber, s);
    }
  }
  chi = block_sum(chi, scratch);
  if (threadIdx.x == 0) d.blk_red[blockIdx.x] = chi;
  if (last_block(&d.st->cnt[7])) {
    const FP s = reduce_partials(d.blk_red, gridDim.x, scratch);
    if (threadIdx.x == 0) {
      if (!d.dist || force)
        d.st->chi2_new = s;
      else
        d.red[red_scalars(d) + kRedChi] = s;
    }
  }
}


// =====================================================================
// Schur-complement solver mode (no reference counterpart: SPEC.md:164,366
// non-goal, PAPER.md:561 future work; CPU statement + dense oracle in
// oracle/restatement.py SchurSystem). Scaled damped system A = D H D + L:
//   S = A_cc - A_cp A_pp^-1 A_pc (cameras), r_c = rhs_c - A_cp A_pp^-1 rhs_p,
//   PCG on S with block-Jacobi of S's camera blocks, x_p by back-substitution.
// Every kernel is a tile pass with the point blocks local to the tile; the
// A_pp^-1 are the point preconditioner blocks (k_precond, exact LLT).
// =====================================================================

// packed 3x3 symmetric (p3 layout) times vector
template <typename T, typename M>
__device__ inline void sym3_mul(const M* m, const T* v, T* out) {
  out[0] = T(m[0]) * v[0] + T(m[1]) * v[1] + T(m[2]) * v[2];
  out[1] = T(m[1]) * v[0] + T(m[3]) * v[1] + T(m[4]) * v[2];
  out[2] = T(m[2]) * v[0] + T(m[4]) * v[1] + T(m[5]) * v[2];
}

// camera blocks of S: per edge E = B A_pp^-1 B^T with B = w Jc~^T Jp~ (9x3)
template <typename FP, typename SP>
__global__ void __launch_bounds__(kTileThreads) k_schur_pre_tiles(Dev<FP, SP> d) {
  if (!d.st->iter_active) return;
  const int tid = threadIdx.x, lane = tid & 31;
  const uint64_t pcol0 = 9ull * d.nc;
  const uint32_t t = blockIdx.x;
  const uint32_t eb = d.tile_ebeg[t], ne_t = d.tile_ecnt[t], pb = d.tile_pbeg[t];
  for (uint32_t c0 = 0; c0 < ne_t; c0 += kTileThreads) {
    const uint32_t j = c0 + tid;
    const bool valid = j < ne_t;
    const uint32_t e = eb + (valid ? j : 0);
    const uint32_t cam = d.d_cam[e];
    const uint64_t pid = pb + d.d_lpt[e];
    const uint64_t pcol = pcol0 + 3 * pid;
    FP jc[18], jp[6];
    {
      arith_t<SP> ja[18], pa[6];
      load_J(d, e, cam, ja, pa);
#pragma unroll
      for (int k = 0; k < 18; ++k) jc[k] = static_cast<FP>(ja[k]) * d.D[9ull * cam + (k % 9)];
#pragma unroll
      for (int k = 0; k < 6; ++k) jp[k] = static_cast<FP>(pa[k]) * d.D[pcol + (k % 3)];
    }
    const FP w = d.w ? d.w[e] : FP(1);
    const bool on = valid && d.col_free[pcol];
    FP B[27], C[27];
#pragma unroll
    for (int i = 0; i < 9; ++i)
#pragma unroll
      for (int k = 0; k < 3; ++k) B[3 * i + k] = on ? w * (jc[i] * jp[k] + jc[9 + i] * jp[3 + k]) : FP(0);
    const FP* M = d.Mp + 6 * pid;
#pragma unroll
    for (int i = 0; i < 9; ++i) sym3_mul<FP, FP>(M, &B[3 * i], &C[3 * i]);
    const uint32_t chunk = d.tile_chunk_base[t] + (c0 + (tid & ~31)) / 32;
    const RunInfo ri = run_info(cam, valid, d.chunk_part_base[chunk]);
#pragma unroll
    for (int g = 0; g < 5; ++g) {
      FP v[9];
#pragma unroll
      for (int k = 0; k < 9; ++k) {
        const int q = 9 * g + k;
        const int a = p9row(q), bb = p9col(q);
        v[k] = C[3 * a] * B[3 * bb] + C[3 * a + 1] * B[3 * bb + 1] + C[3 * a + 2] * B[3 * bb + 2];
      }
      seg_reduce<FP, 9>(v, lane, ri.run_end);
      if (ri.head) {
        FP* dst = d.part + static_cast<uint64_t>(d.run_slot[ri.slot]) * kLinVals + 9 * g;
#pragma unroll
        for (int k = 0; k < 9; ++k) dst[k] = v[k];
      }
    }
  }
}

// S_c = D H_cc D + L - sum(E), LLT inverse -> Mc (fallback like k_precond)
template <typename FP, typename SP>
__global__ void k_schur_pre_cams(Dev<FP, SP> d) {
  if (!d.st->iter_active) return;
  const uint64_t c = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (c >= d.nc) return;
  const uint64_t col = 9 * c;
  FP* Mo = d.Mc + 45 * c;
  if (!d.col_free[col]) {
    for (int k = 0; k < 45; ++k) Mo[k] = FP(0);
    return;
  }
  const FP lam = d.st->lambda_solve;
  FP Dv[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) Dv[k] = d.D[col + k];
  FP B[45];
  int q = 0;
#pragma unroll
  for (int i = 0; i < 9; ++i)
#pragma unroll
    for (int j = i; j < 9; ++j, ++q) {
      B[q] = Dv[i] * d.Hc[45 * c + q] * Dv[j];
      if (i == j) B[q] += d.st->before_scaling ? lam * Dv[i] * Dv[i] : lam;
    }
  for (uint32_t s2 = d.cam_part_off[c]; s2 < d.cam_part_off[c + 1]; ++s2) {
    const FP* src = d.part + static_cast<uint64_t>(s2) * kLinVals;  // camera-major storage
#pragma unroll
    for (int k = 0; k < 45; ++k) B[k] -= src[k];
  }
  FP out[45];
  if (!chol_inverse<FP, 9>(B, out)) {
    q = 0;
#pragma unroll
    for (int i = 0; i < 9; ++i)
#pragma unroll
      for (int j = i; j < 9; ++j, ++q) out[q] = (i == j) ? FP(1) / clampv(B[q], FP(d.st->clamp_min), FP(d.st->clamp_max)) : FP(0);
    atomicAdd(&d.st->fallbacks, 1);
  }
#pragma unroll
  for (int k = 0; k < 45; ++k) Mo[k] = out[k];
}

// Shared tile pass: phase 1 y_p = sum_e Jp~^T w Jc~ v_c (points, in SMEM).
// mode 0 (S v): z_p = A_pp^-1 y_p, then per edge g = Jc~^T w (Jc~ v - Jp~ z).
// mode 1 (rhs): z_p = A_pp^-1 rhs_p (no phase 1), g = Jc~^T w Jp~ z.
// mode 2 (back-substitution): x_p = A_pp^-1 (rhs_p - y_p) -> xp (no phase 2).
// vt holds (Arith) D * v for the camera columns.
template <typename FP, typename SP, int MODE>
__global__ void __launch_bounds__(kTileThreads) k_schur_tiles(Dev<FP, SP> d) {
  using A = arith_t<SP>;
  if (!d.st->iter_active) return;
  if (MODE == 0 && d.st->pcg_done) return;
  __shared__ A stage[kTileEdges * 3];
  __shared__ A usm[kTileEdges * 2];
  __shared__ A zt[kTilePoints * 3];
  __shared__ A hacc[3];
  const int tid = threadIdx.x, lane = tid & 31;
  const uint64_t pcol0 = 9ull * d.nc;
  const uint32_t t = blockIdx.x;
  const uint32_t eb = d.tile_ebeg[t], ne_t = d.tile_ecnt[t];
  const uint32_t pb = d.tile_pbeg[t], npt = d.tile_pbeg[t + 1] - pb;
  const bool heavy = ne_t > static_cast<uint32_t>(kTileEdges);
  if (tid < 3) hacc[tid] = A(0);
  __syncthreads();
  if (MODE != 1) {  // phase 1: y_p
    for (uint32_t c0 = 0; c0 < ne_t; c0 += kTileThreads) {
      const uint32_t j = c0 + tid;
      const bool valid = j < ne_t;
      const uint32_t e = eb + (valid ? j : 0);
      const uint32_t cam = d.d_cam[e];
      A jc[18], jp[6];
      load_J(d, e, cam, jc, jp);
      const A* cv = d.vt + 9ull * cam;
      A u0 = A(0), u1 = A(0);
#pragma unroll
      for (int k = 0; k < 9; ++k) {
        u0 += jc[k] * cv[k];
        u1 += jc[9 + k] * cv[k];
      }
      const A wgt = d.w ? static_cast<A>(d.w[e]) : A(1);
      const A q0 = valid ? wgt * u0 : A(0), q1 = valid ? wgt * u1 : A(0);
      if (!heavy && valid) {
        usm[2 * j] = u0;
        usm[2 * j + 1] = u1;
      }
      A h[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) h[k] = jp[k] * q0 + jp[3 + k] * q1;
      if (!heavy) {
        if (valid)
#pragma unroll
          for (int k = 0; k < 3; ++k) stage[j * 3 + k] = h[k];
      } else {
#pragma unroll
        for (int k = 0; k < 3; ++k) stage[tid * 3 + k] = h[k];
        __syncthreads();
        if (tid < 3) {
          A acc = hacc[tid];
          const uint32_t nvalid = min(static_cast<uint32_t>(kTileThreads), ne_t - c0);
          for (uint32_t q = 0; q < nvalid; ++q) acc += stage[q * 3 + tid];
          hacc[tid] = acc;
        }
        __syncthreads();
      }
    }
    __syncthreads();
  }
  // per point: z (modes 0, 1) or x_p (mode 2)
  for (uint32_t i = tid; i < npt; i += blockDim.x) {
    const uint64_t pid = pb + i;
    const uint64_t col = pcol0 + 3 * pid;
    const bool freev = d.col_free[col];
    FP y[3] = {FP(0), FP(0), FP(0)};
    if (MODE != 1) {
      A acc[3];
      if (heavy) {
#pragma unroll
        for (int k = 0; k < 3; ++k) acc[k] = hacc[k];
      } else {
        acc[0] = acc[1] = acc[2] = A(0);
        for (uint32_t q = d.pt_slot_off[pid]; q < d.pt_slot_off[pid + 1]; ++q) {
          const uint32_t sl = d.pt_slots[q];
#pragma unroll
          for (int k = 0; k < 3; ++k) acc[k] += stage[sl * 3 + k];
        }
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) y[k] = d.D[col + k] * static_cast<FP>(acc[k]);  // Jp~^T = D_p Jp^T
    }
    FP rhs[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) rhs[k] = -d.D[col + k] * d.b[col + k];
    FP src[3], z[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) src[k] = MODE == 0 ? y[k] : (MODE == 1 ? rhs[k] : rhs[k] - y[k]);
    sym3_mul<FP, FP>(d.Mp + 6 * pid, src, z);
    if (MODE == 2) {
#pragma unroll
      for (int k = 0; k < 3; ++k) d.xp[3 * pid + k] = freev ? z[k] : FP(0);
    } else {
#pragma unroll
      for (int k = 0; k < 3; ++k) zt[3 * i + k] = freev ? static_cast<A>(d.D[col + k] * z[k]) : A(0);
    }
  }
  if (MODE == 2) return;
  __syncthreads();
  // phase 2: camera contributions
  for (uint32_t c0 = 0; c0 < ne_t; c0 += kTileThreads) {
    const uint32_t j = c0 + tid;
    const bool valid = j < ne_t;
    const uint32_t e = eb + (valid ? j : 0);
    const uint32_t cam = d.d_cam[e];
    const uint32_t lp = d.d_lpt[e];
    A jc[18], jp[6];
    load_J(d, e, cam, jc, jp);
    A u0 = A(0), u1 = A(0);
    if (MODE == 0) {
      if (!heavy) {
        u0 = usm[2 * j];
        u1 = usm[2 * j + 1];
      } else {
        const A* cv = d.vt + 9ull * cam;
#pragma unroll
        for (int k = 0; k < 9; ++k) {
          u0 += jc[k] * cv[k];
          u1 += jc[9 + k] * cv[k];
        }
      }
    }
    A v0 = A(0), v1 = A(0);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      v0 += jp[k] * zt[3 * lp + k];
      v1 += jp[3 + k] * zt[3 * lp + k];
    }
    const A wgt = d.w ? static_cast<A>(d.w[e]) : A(1);
    const A q0 = valid ? wgt * (MODE == 0 ? u0 - v0 : v0) : A(0);
    const A q1 = valid ? wgt * (MODE == 0 ? u1 - v1 : v1) : A(0);
    A g[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) g[k] = jc[k] * q0 + jc[9 + k] * q1;
    const uint32_t chunk = d.tile_chunk_base[t] + (c0 + (tid & ~31)) / 32;
    const RunInfo ri = run_info(cam, valid, d.chunk_part_base[chunk]);
    seg_reduce<A, 9>(g, lane, ri.run_end);
    if (ri.head) {
      FP* dst = d.part + static_cast<uint64_t>(d.run_slot[ri.slot]) * 9;
#pragma unroll
      for (int k = 0; k < 9; ++k) dst[k] = static_cast<FP>(g[k]);
    }
  }
  if (MODE == 0 && tid < 8) d.tile_red[8ull * t + tid] = FP(0);  // no point columns in the Schur PCG
}

// r_c = rhs_c - D_c * sum(partials)
template <typename FP, typename SP>
__global__ void __launch_bounds__(32 * kCamWarps) k_schur_rhs_cams(Dev<FP, SP> d) {
  if (!d.st->iter_active) return;
  const int lane = threadIdx.x & 31;
  const uint32_t c = blockIdx.x * kCamWarps + (threadIdx.x >> 5);
  if (c >= d.nc) return;
  FP acc[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) acc[k] = FP(0);
  for (uint32_t q = d.cam_part_off[c] + lane; q < d.cam_part_off[c + 1]; q += 32) {
    const FP* src = d.part + static_cast<uint64_t>(q) * 9;  // camera-major storage
#pragma unroll
    for (int k = 0; k < 9; ++k) acc[k] += src[k];
  }
#pragma unroll
  for (int k = 0; k < 9; ++k) acc[k] = warp_sum(acc[k]);
  if (lane < 9) {
    const uint64_t col = 9ull * c + lane;
    FP a = acc[0];
#pragma unroll
    for (int k = 1; k < 9; ++k)
      if (lane == k) a = acc[k];
    d.rc[col] = d.col_free[col] ? -d.D[col] * d.b[col] - d.D[col] * a : FP(0);
  }
}

// vt (cameras) = D * x_c after the Schur PCG (x_c unscaled), for back-substitution
template <typename FP, typename SP>
__global__ void k_schur_xc(Dev<FP, SP> d) {
  using A = arith_t<SP>;
  if (!d.st->iter_active) return;
  const FP unscale = d.st->unscale;
  const bool zero = d.st->pcg_zero;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < 9ull * d.nc;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    d.vt[i] = static_cast<A>(d.D[i] * (zero ? FP(0) : widen<FP>(d.xs[i]) * unscale));
}

// Accept / reject, Nielsen damping, termination, per-iteration record
// (levenberg_marquardt.hpp:171-220, update_damping :88-98). One thread.
template <typename FP>
__global__ void k_decide(State<FP>* st, gb_iteration_record* recs) {
  if (!st->iter_active) return;
  gb_iteration_record& rec = recs[st->lm_it - 1];
  rec.pcg_iterations = st->pcg_it;
  rec.pcg_converged = st->pcg_conv;
  rec.pcg_relative_residual = st->pcg_relres;
  rec.precond_fallback_blocks = st->fallbacks;
  FP lambda = st->lambda, nu = st->nu;
  if (st->use_guard && !st->pcg_conv && st->pcg_relres > st->pcg_ratio * st->pcg_tol) {
    rec.low_quality_step = 1;
    lambda *= nu;
  }
  const FP chi2 = st->chi2;
  const FP chi2_new = st->step_finite ? st->chi2_new : FP(NAN);
  rec.chi2_after = static_cast<double>(chi2_new);
  const bool accepted = is_finite(chi2_new) && chi2_new < chi2;
  rec.accepted = accepted ? 1 : 0;
  st->accepted = accepted ? 1 : 0;
  FP rel = FP(0);
  if (accepted) {
    st->accepted_steps += 1;
    const FP gain = st->pred > FP(0) ? (chi2 - chi2_new) / st->pred : FP(INFINITY);
    const FP g = FP(2) * gain - FP(1);
    lambda *= fmax(FP(1) / FP(3), FP(1) - g * g * g);
    nu = FP(2);
    rel = (chi2 - chi2_new) / chi2;
    st->chi2 = chi2_new;  // == LinearSystem::linearize() at the accepted point
    st->do_linearize = 1;
  } else {
    lambda *= nu;
    nu *= FP(2);
    st->do_linearize = st->refresh_on_reject;
  }
  st->lambda = lambda;
  st->nu = nu;
  st->rel_decrease = rel;
  if (accepted && static_cast<double>(rel) < st->tol) {
    st->termination = GB_TERM_TOLERANCE_REACHED;
    st->terminated = 1;
  } else if (static_cast<double>(lambda) > st->lambda_max) {
    st->termination = GB_TERM_DAMPING_OVERFLOW;
    st->terminated = 1;
  } else if (st->lm_it >= st->max_iterations) {
    st->termination = GB_TERM_MAX_ITERATIONS;
    st->terminated = 1;
  }
  if (st->terminated) st->do_linearize = 0;  // the refreshed linearization is never observed
}

// Accepted step becomes the current point (the reference mutates in place and
// restores the snapshot on reject, graph.hpp:114-128; here the candidate
// lives in x_new and is copied on accept, so restore is a no-op).
template <typename FP, typename SP>
__global__ void k_commit(Dev<FP, SP> d) {
  if (!d.st->iter_active || !d.st->accepted) return;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < d.ncols;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    d.x[i] = d.x_new[i];
}

}  // namespace gb
