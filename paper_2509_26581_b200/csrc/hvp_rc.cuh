// Recompute HVP: the matrix-free Hessian-vector product of the analytic
// Snavely factor without a Jacobian store (LinearSystem::hvp,
// linear_system.hpp:104-115; hvp_forward factor_descriptor.hpp:372-407,
// hvp_scatter :409-433, evaluated like the low-memory path :673-684).
//
// Analytic mode with SP == FP (fp64, fp32) and dynamic mode in any precision
// (J at FP, cast to Arith, factor_descriptor.hpp:673-684; for fp32-bf16 only
// the PCG vectors are bf16, widened on load and narrowed on store). The stored
// operator J = [U·Dw | U | dist p, f n p, f n^2 p ; U R] (snavely.hpp:103-153)
// is applied in its factored form, with every per-camera product hoisted out
// of the edge loop:
//   forward   u = U (M X + v_t + R v_p) + p (dist v_f + n (f v_k1 + n f v_k2)),
//             M = [Dw(e_0) v_w | Dw(e_1) v_w | Dw(e_2) v_w]  (Dw is linear in X),
//   scatter   q = w u, h = U^T q:  point  J_p^T q = R^T h;
//             camera J_c^T q = [sum_k,i T_k(i,.) X_k h_i | h | dist p.q, f n p.q, f n^2 p.q],
// so an edge needs only its point X, its point's D p, and 30 per-camera values
// it shares with its neighbours, and a camera run accumulates 15 values
// (X h^T, h, three intrinsic scalars) that the camera kernel contracts with
// T_k = Dw(e_k) once per camera. Nothing per edge is read from HBM except
// two 16-bit indices (and the Huber weight): the HVP moves ~0.9 GB at
// Final-13682 fp64 instead of the 4.7 GB of the factored J store, and
// linearize no longer writes a Jacobian.
//
// Kernel shape (k_hvp_rc): one persistent CTA per SM, a producer warp that
// streams each normal tile (static aux blob, per-linearization lin blob with
// D and the tile cameras' [R t f k1 k2], the tile's points X and p (+ z when
// the direction update is pending), the tile cameras' per-HVP records
// [M v_t v_int]) into a 2-stage shared-memory ring with cp.async.bulk; a
// preparer warp (p = z + beta p, v_p = D p); 8 consumer warps with TWO edges
// per thread (one camera load serves both when they share a camera, as ~98 %
// of pairs do), camera sums in registers, one 15-value partial per thread
// pair in shared memory; after one named barrier half the consumers sum the
// camera runs (one thread per (camera, value)) while the other half sums the
// points from their slot lists, alternating by tile.
#pragma once

#include <algorithm>

#include "hvp_pipe.cuh"

namespace gb {

constexpr int kRcVals = 15;  // camera-run partial: S(k, i) = X_k h_i (9), h (3), dist p.q, n p.q, n^2 p.q

// Shared memory: a byte ring of tile regions (each tile's inputs at their
// exact size, so ~10 typical tiles are in flight: the stream is latency-bound
// per tile, not bandwidth-bound) and one work buffer per consumer group
// (per-thread camera-run partials, odd-start run partials, per-edge point
// contributions, run starts). A tile region: [header | aux blob | lin blob |
// p | z (direction update pending) | tile camera records].
constexpr int kRcGroups = 2;                    // consumer groups, alternating tiles
constexpr int kRcEdgesPerThread = 4;            // contiguous edges of one thread
constexpr int kRcGroupThreads = kTileEdges / kRcEdgesPerThread;  // 128
constexpr int kRcAStr = kSegSlots + 1;          // row stride of the per-segment partials (odd: distinct banks)
constexpr int kRcGpStr = kTileEdges + 4;        // row stride of the per-edge point contributions
constexpr int kRcSlots = 16;                    // max tiles in flight per CTA
constexpr uint32_t kRcHdrBytes = 64;

struct RcLayout {
  uint32_t A, gp, work_bytes;
  uint32_t ring, ring_bytes, slots, bars, total_bytes;
  uint32_t max_region;  // largest tile region (a tile never needs more)
  int dbg;  // experiments only (GB_RC_DBG): 1 skip the edge math, 2 skip the epilogue, 8 per-role wait cycles,
           // 16 utility warps wait with the suspend hint instead of the nanosleep back-off
  unsigned long long* prof;  // [8] (dbg & 8): cycles waiting / total per role, summed over CTAs
};

template <typename FP>
inline RcLayout rc_layout(bool huber, uint32_t smem_budget) {
  RcLayout L{};
  uint32_t o = 0;
  auto take = [&](uint64_t bytes) {
    const uint32_t r = o;
    o += r16(bytes);
    return r;
  };
  L.A = take(static_cast<uint64_t>(kRcVals) * kRcAStr * sizeof(FP));
  L.gp = take(3ull * kRcGpStr * sizeof(FP));
  L.work_bytes = o;
  L.max_region = kRcHdrBytes + aux_sections(kTileEdges, kTilePoints).bytes +
                 rc_lin_sections<FP>(kTileEdges, kTilePoints, kTileCams, huber).bytes +
                 4 * r16(kTilePoints * 3 * sizeof(FP) + 16) + kTileCams * kRcRec * sizeof(FP) + 128;
  L.slots = 2 * kRcGroups * L.work_bytes;  // two work buffers per group (alternating tiles)
  L.bars = L.slots + 4 * kRcSlots;
  L.ring = L.bars + 4 * kRcSlots * 8;
  L.ring = (L.ring + 127) / 128 * 128;
  L.ring_bytes = smem_budget > L.ring ? (smem_budget - L.ring) / 128 * 128 : 0;
  L.total_bytes = L.ring + L.ring_bytes;
  return L;
}

enum RcHdr : int { kRT = 0, kRNe, kRNpt, kRNcam, kRPb, kRCb, kRDp, kRDz, kROAux, kROLin, kROP, kROZ, kROTc, kROV, kROX,
                   kRCount };

// mbar_wait that sleeps (suspend-time hint) instead of spinning, and adds its
// waiting cycles to acc when profiling
__device__ __forceinline__ void mbar_sleep_wait(uint64_t* bar, unsigned parity) {
#ifdef GB_RC_SPIN
  mbar_wait(bar, parity);
  return;
#endif
  asm volatile(
      "{\n .reg .pred P;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1, %2;\n"
      " @!P bra WAIT_%=;\n}" ::"r"(smem_addr(bar)),
      "r"(parity), "r"(1000000)
      : "memory");
}
// utility-warp wait: non-blocking probes with an exponential nanosleep
// back-off (32 -> 512 ns), so a waiting producer / loader / preparer does not
// keep issuing probe instructions on an SMSP it shares with consumer warps
__device__ __forceinline__ bool mbar_test(uint64_t* bar, unsigned parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred P;\n mbarrier.test_wait.parity.shared::cta.b64 P, [%1], %2;\n selp.u32 %0, 1, 0, P;\n}"
      : "=r"(ok)
      : "r"(smem_addr(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_backoff_wait(uint64_t* bar, unsigned parity, bool backoff) {
  if (!backoff) {
    mbar_sleep_wait(bar, parity);
    return;
  }
  unsigned ns = 32;  // measured: caps of 256 / 2048 ns were slower than 512
  while (!mbar_test(bar, parity)) {
    __nanosleep(ns);
    ns = ns < 512u ? 2 * ns : 512u;
  }
}
__device__ __forceinline__ void mbar_wait_u(uint64_t* bar, unsigned parity, bool backoff, bool on,
                                            unsigned long long& acc) {
  const long long t0 = on ? clock64() : 0;
  mbar_backoff_wait(bar, parity, backoff);
  if (on) acc += static_cast<unsigned long long>(clock64() - t0);
}
__device__ __forceinline__ void mbar_wait_t(uint64_t* bar, unsigned parity, bool on, unsigned long long& acc) {
  if (!on) {
    mbar_sleep_wait(bar, parity);
    return;
  }
  const long long t0 = clock64();
  mbar_sleep_wait(bar, parity);
  acc += static_cast<unsigned long long>(clock64() - t0);
}


// dP/dw of the analytic chain at a point x (snavely.hpp:103-121; the same
// expression as snavely_linearize's Dw): linear in x.
template <typename FP>
__device__ inline void rot_jacobian(const FP* w, FP s, FP c, FP s1, FP c2, const FP* x, FP* Dw) {
  const FP cr[3] = {w[1] * x[2] - w[2] * x[1], w[2] * x[0] - w[0] * x[2], w[0] * x[1] - w[1] * x[0]};
  const FP dt = w[0] * x[0] + w[1] * x[1] + w[2] * x[2];
  const FP skx[9] = {FP(0), -x[2], x[1], x[2], FP(0), -x[0], -x[1], x[0], FP(0)};
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      Dw[3 * i + j] = -s * x[i] * w[j] + s1 * cr[i] * w[j] - s * skx[3 * i + j] + c2 * dt * w[i] * w[j] +
                      c * (w[i] * x[j] + (i == j ? dt : FP(0)));
}

// T_k = Dw(e_k) of camera c (its angle-axis from params, chain coefficients
// from its camera_pre record)
template <typename FP>
__device__ inline void rot_basis(const FP* cam, const FP* pre, FP (&T)[3][9]) {
  const FP w[3] = {cam[0], cam[1], cam[2]};
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const FP e[3] = {FP(k == 0), FP(k == 1), FP(k == 2)};
    rot_jacobian<FP>(w, pre[4], pre[5], pre[6], pre[7], e, T[k]);
  }
}

// per-camera values an edge needs (30, in registers for both edges of a pair)
template <typename FP>
struct RcCam {
  FP R[9], t[3], f, k1, k2;        // static (per linearization)
  FP M[9], vt[3], vf, vk1, vk2;    // per HVP: M, v_t, v_f, f v_k1, f v_k2
};

template <typename FP>
__device__ __forceinline__ void rc_load_cam(const FP* scam, const FP* stc, uint32_t lc, RcCam<FP>& C) {
  FP a[kRcRec], b[kRcRec];
  load16<FP, kRcRec>(scam + kRcRec * lc, a);
  load16<FP, kRcRec>(stc + kRcRec * lc, b);
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    C.R[k] = a[k];
    C.M[k] = b[k];
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    C.t[k] = a[9 + k];
    C.vt[k] = b[9 + k];
  }
  C.f = a[12];
  C.k1 = a[13];
  C.k2 = a[14];
  C.vf = b[12];
  C.vk1 = b[13];
  C.vk2 = b[14];
}

// 1/x: IEEE division in fp32; in fp64 the MUFU seed (rcp.approx.ftz.f64,
// ~2^-23) refined by one third-order step r (1 + e + e^2), e = 1 - x r (relative
// error ~2^-69, i.e. rounding level; no slow-path branch)
__device__ __forceinline__ float rc_rcp(float x) { return 1.0f / x; }
__device__ __forceinline__ double rc_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);  // one Newton step with the quadratic term: error ~ e^3
  return fma(r, fma(e, e, e), r);
}

// One edge: the forward product and the scatter terms, with U = du/dP
// written as -1/P_z [A00 A01 m0; A01 A11 m1] (snavely.hpp:130-148) so it is
// never formed: h = U^T q, the intrinsic scalars (dist, n, n^2) * p.q and the
// point contribution R^T h. Invalid edges yield exact zeros.
template <typename FP>
struct RcEdge {
  FP h[3], a[3], g[3];
};
template <typename FP, bool HUBER>
__device__ __forceinline__ RcEdge<FP> rc_edge(const RcCam<FP>& C, const FP* X, const FP* vp, FP wgt, bool valid) {
  FP P[3], y[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    P[i] = fma(C.R[3 * i + 2], X[2], fma(C.R[3 * i + 1], X[1], fma(C.R[3 * i], X[0], C.t[i])));
    y[i] = fma(C.M[3 * i + 2], X[2],
               fma(C.M[3 * i + 1], X[1],
                   fma(C.M[3 * i], X[0], fma(C.R[3 * i + 2], vp[2], fma(C.R[3 * i + 1], vp[1], fma(C.R[3 * i], vp[0], C.vt[i]))))));
  }
  const FP iz = rc_rcp(P[2]);
  const FP p0 = -P[0] * iz, p1 = -P[1] * iz;
  const FP n = fma(p0, p0, p1 * p1);
  const FP dist = fma(n, fma(n, C.k2, C.k1), FP(1));
  const FP gg = FP(2) * fma(FP(2) * C.k2, n, C.k1);
  const FP gp0 = gg * p0, gp1 = gg * p1;
  const FP A00 = C.f * fma(gp0, p0, dist), A01 = C.f * (gp0 * p1), A11 = C.f * fma(gp1, p1, dist);
  const FP m0 = fma(A00, p0, A01 * p1), m1 = fma(A01, p0, A11 * p1);
  const FP s = fma(n, fma(n, C.vk2, C.vk1), dist * C.vf);
  const FP Ay0 = fma(m0, y[2], fma(A01, y[1], A00 * y[0]));
  const FP Ay1 = fma(m1, y[2], fma(A11, y[1], A01 * y[0]));
  FP q0 = fma(-iz, Ay0, p0 * s), q1 = fma(-iz, Ay1, p1 * s);
  if (HUBER) {
    q0 *= wgt;
    q1 *= wgt;
  }
  const FP qq0 = -iz * q0, qq1 = -iz * q1;
  RcEdge<FP> o;
  o.h[0] = valid ? fma(A01, qq1, A00 * qq0) : FP(0);
  o.h[1] = valid ? fma(A11, qq1, A01 * qq0) : FP(0);
  o.h[2] = valid ? fma(m1, qq1, m0 * qq0) : FP(0);
  const FP pq = fma(p1, q1, p0 * q0);
  o.a[0] = valid ? dist * pq : FP(0);
  o.a[1] = valid ? n * pq : FP(0);
  o.a[2] = valid ? n * (n * pq) : FP(0);
#pragma unroll
  for (int k = 0; k < 3; ++k) o.g[k] = fma(C.R[6 + k], o.h[2], fma(C.R[3 + k], o.h[1], C.R[k] * o.h[0]));
  return o;
}

__device__ __forceinline__ void rc_setmaxnreg_inc216() { asm volatile("setmaxnreg.inc.sync.aligned.u32 208;\n" ::: "memory"); }
__device__ __forceinline__ void rc_setmaxnreg_dec56() { asm volatile("setmaxnreg.dec.sync.aligned.u32 72;\n" ::: "memory"); }

// the 15 camera-run values of one edge added into acc (S(k, i) = X_k h_i, h, a)
template <typename FP>
__device__ __forceinline__ void rc_accumulate(const RcEdge<FP>& o, const FP* X, FP (&acc)[kRcVals]) {
#pragma unroll
  for (int k = 0; k < 3; ++k)
#pragma unroll
    for (int i = 0; i < 3; ++i) acc[3 * k + i] = fma(X[k], o.h[i], acc[3 * k + i]);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    acc[9 + i] += o.h[i];
    acc[12 + i] += o.a[i];
  }
}

// Warp roles (384 threads, one CTA per SM):
//   warps 0-3, 4-7   consumer groups 0 and 1 (208 registers): group g takes
//                    the CTA's tiles it = g, g + 2, ...; thread i of a group
//                    owns tile edges 4i .. 4i + 3 (one camera load serves all
//                    of them unless a run starts inside), then the group's
//                    epilogue (camera runs, points) after a group barrier
//   warp 8           producer (ring regions, headers, one bulk copy of the tile blob)
//   warp 9           preparer (p = z + beta p, v_p = D p)
//   warp 10          loader (p, z, tile camera records by cp.async)
constexpr int kRcThreadsWS = 384;

template <typename FP, typename SP, bool HUBER>
__global__ void __launch_bounds__(kRcThreadsWS, 1) k_hvp_rc(Dev<FP, SP> d, RcLayout L) {
  if (!d.st->iter_active || d.st->pcg_done) return;
  extern __shared__ __align__(128) unsigned char rc_smem[];
  uint32_t* slot_off = reinterpret_cast<uint32_t*>(rc_smem + L.slots);
  uint64_t* full = reinterpret_cast<uint64_t*>(rc_smem + L.bars);
  uint64_t* empty = full + kRcSlots;
  uint64_t* ready = empty + kRcSlots;
  uint64_t* blob = ready + kRcSlots;  // the tile blob's bulk copy (producer) has landed
  unsigned char* ring = rc_smem + L.ring;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < kRcSlots; ++s) {
      mbar_init(&full[s], 32);  // every loader lane's cp.async group (p, z, camera records)
      mbar_init(&empty[s], kRcGroupThreads / 32);  // the owning group's warps
      mbar_init(&ready[s], 32);
      mbar_init(&blob[s], 1);  // producer lane 0: arrive + bulk tx
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint64_t pcol0 = 9ull * d.nc;
  const uint32_t ntiles = d.n_normal;
  const bool dir = d.st->dir_pending != 0;
  const bool xpend = d.st->x_pending != 0;  // x += alpha p of the last PCG update (preparer, on the loaded p)
  const bool pf = (L.dbg & 8) && lane == 0;
  const bool bo = !(L.dbg & 16);  // utility warps poll with a nanosleep back-off (GB_RC_DBG & 16: suspend-hint waits)

  if (warp < 2 * kRcGroupThreads / 32) {
    rc_setmaxnreg_inc216();
    // ---------------------------------------------------------- consumer groups
    const uint32_t g = static_cast<uint32_t>(warp) / (kRcGroupThreads / 32);
    const uint32_t gt = static_cast<uint32_t>(tid) - g * kRcGroupThreads;  // 0..127
    const FP lam = static_cast<FP>(d.st->lambda_solve);
    const int before = d.st->before_scaling;
    unsigned long long w_ready = 0;
    const long long t_start = clock64();
    for (uint32_t it = g, k2 = 0;; it += kRcGroups, ++k2) {
      // the group's two work buffers alternate: the edge phase of tile k2 + 1
      // writes one while no thread can still read it (every thread passed the
      // barrier of tile k2 only after finishing the epilogue of tile k2 - 1)
      unsigned char* wk = rc_smem + (2 * g + (k2 & 1u)) * L.work_bytes;
      FP* sA = reinterpret_cast<FP*>(wk + L.A);
      FP* gp = reinterpret_cast<FP*>(wk + L.gp);
      if (blockIdx.x + it * gridDim.x >= ntiles) break;
      const int s = static_cast<int>(it % kRcSlots);
      mbar_wait_t(&ready[s], (it / kRcSlots) & 1u, pf, w_ready);
      const unsigned char* rg = ring + slot_off[s];
      const uint32_t* h = reinterpret_cast<const uint32_t*>(rg);
      const uint32_t ne = h[kRNe], npt = h[kRNpt], ncam = h[kRNcam];
      const AuxSec as = aux_sections(ne, npt);
      const RcLinSec ls = rc_lin_sections<FP>(ne, npt, ncam, HUBER);
      const unsigned char* aux = rg + h[kROAux];
      const unsigned char* lin = rg + h[kROLin];
      // ---- edge phase: thread gt = run-aligned segment gt (<= 8 edges of one camera)
      const uint16_t* segs = reinterpret_cast<const uint16_t*>(aux + as.seg);
      const uint32_t sg = segs[gt], e0 = sg & 511u, cnt = sg >> 9;
      if (!(L.dbg & 1) && cnt) {
        const uint16_t* slc = reinterpret_cast<const uint16_t*>(aux + as.lcam);
        const uint16_t* slp = reinterpret_cast<const uint16_t*>(aux + as.lpt);
        const FP* sX = reinterpret_cast<const FP*>(lin + ls.X);
        const FP* svp = reinterpret_cast<const FP*>(rg + h[kROV]);
        const FP* scam = reinterpret_cast<const FP*>(lin + ls.cam);
        const FP* stc = reinterpret_cast<const FP*>(rg + h[kROTc]);
        const FP* sw = reinterpret_cast<const FP*>(lin + ls.w);
        const uint16_t* spos = reinterpret_cast<const uint16_t*>(aux + as.pos);
        RcCam<FP> C;
        rc_load_cam<FP>(scam, stc, slc[e0], C);
        FP acc[kRcVals];
#pragma unroll
        for (int v = 0; v < kRcVals; ++v) acc[v] = FP(0);
        uint32_t k = 0;
        for (; k + 1 < cnt; k += 2) {  // two edges per step: independent chains
          const uint32_t ea = e0 + k, eb = ea + 1;
          const uint32_t la = slp[ea], lb = slp[eb];
          const FP Xa[3] = {sX[3 * la], sX[3 * la + 1], sX[3 * la + 2]};
          const FP Va[3] = {svp[3 * la], svp[3 * la + 1], svp[3 * la + 2]};
          const FP Xb[3] = {sX[3 * lb], sX[3 * lb + 1], sX[3 * lb + 2]};
          const FP Vb[3] = {svp[3 * lb], svp[3 * lb + 1], svp[3 * lb + 2]};
          const FP wa = HUBER ? sw[ea] : FP(1), wb = HUBER ? sw[eb] : FP(1);
          const RcEdge<FP> oa = rc_edge<FP, HUBER>(C, Xa, Va, wa, true);
          const RcEdge<FP> ob = rc_edge<FP, HUBER>(C, Xb, Vb, wb, true);
          rc_accumulate<FP>(oa, Xa, acc);
          rc_accumulate<FP>(ob, Xb, acc);
          const uint32_t pa = spos[ea], pbb = spos[eb];  // point-slot order: each point's contributions contiguous
#pragma unroll
          for (int q = 0; q < 3; ++q) {
            gp[q * kRcGpStr + pa] = oa.g[q];
            gp[q * kRcGpStr + pbb] = ob.g[q];
          }
        }
        if (k < cnt) {  // odd tail
          const uint32_t ea = e0 + k, la = slp[ea];
          const FP Xa[3] = {sX[3 * la], sX[3 * la + 1], sX[3 * la + 2]};
          const FP Va[3] = {svp[3 * la], svp[3 * la + 1], svp[3 * la + 2]};
          const FP wa = HUBER ? sw[ea] : FP(1);
          const RcEdge<FP> oa = rc_edge<FP, HUBER>(C, Xa, Va, wa, true);
          rc_accumulate<FP>(oa, Xa, acc);
          const uint32_t pa = spos[ea];
#pragma unroll
          for (int q = 0; q < 3; ++q) gp[q * kRcGpStr + pa] = oa.g[q];
        }
#pragma unroll
        for (int v = 0; v < kRcVals; ++v) sA[v * kRcAStr + gt] = acc[v];
      }
      asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "n"(kRcGroupThreads) : "memory");
      // ---- epilogue, one item per thread: camera-run values (camera lc,
      // value v: segments [rseg[lc], rseg[lc + 1]) in segment order) first,
      // then points (contiguous point-slot ranges); one pass mixes the tail of
      // the first kind with the head of the second
      const uint32_t cb = h[kRCb];
      const uint16_t* rseg = reinterpret_cast<const uint16_t*>(aux + as.rseg);
      const uint16_t* spso = reinterpret_cast<const uint16_t*>(aux + as.pso);
      const uint8_t* scf = aux + as.cf;
      const FP* sD = reinterpret_cast<const FP*>(lin + ls.D);
      const SP* sp = reinterpret_cast<const SP*>(rg + h[kROP] + h[kRDp]);
      const uint32_t pb = h[kRPb];
      constexpr uint32_t kVG = 5;  // values per camera item: 3 items per camera, so a tile's camera
                                   // items and points usually fit one pass of the group's 128 threads
      const uint32_t ncv = (kRcVals / kVG) * ncam;
      FP dot = FP(0);
      for (uint32_t o = gt; o < ncv + npt && !(L.dbg & 2); o += kRcGroupThreads) {
        if (o < ncv) {
          const uint32_t lc = o / (kRcVals / kVG), v0 = kVG * (o - (kRcVals / kVG) * lc);
          const FP* src = sA + v0 * kRcAStr;
          FP a[kVG];
#pragma unroll
          for (int u = 0; u < static_cast<int>(kVG); ++u) a[u] = FP(0);
          const uint32_t qe = rseg[lc + 1];
          for (uint32_t q = rseg[lc]; q < qe; ++q)
#pragma unroll
            for (int u = 0; u < static_cast<int>(kVG); ++u) a[u] += src[u * kRcAStr + q];
#pragma unroll
          for (int u = 0; u < static_cast<int>(kVG); ++u)
            d.part15[static_cast<uint64_t>(kRcRec) * (cb + lc) + v0 + u] = a[u];
        } else {
          const uint32_t pi = o - ncv;
          FP a[3] = {FP(0), FP(0), FP(0)};
          const uint32_t q0 = spso[pi], q1 = spso[pi + 1];
#pragma unroll 4
          for (uint32_t q = q0; q < q1; ++q)  // contiguous: the edges wrote in slot order
#pragma unroll
            for (int k = 0; k < 3; ++k) a[k] += gp[k * kRcGpStr + q];
          const uint64_t col = pcol0 + 3ull * (pb + pi);
          const bool freev = scf[3 * pi];
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            const FP Dk = sD[3 * pi + k];
            const FP damp = before ? lam * Dk * Dk : lam;
            const SP pk = sp[3 * pi + k];
            if (dir) d.p[col + k] = pk;
            const FP pw = widen<FP>(pk);
            const FP out = freev ? damp * pw + Dk * a[k] : FP(0);
            const SP os = narrow<SP>(out);
            d.ap[col + k] = os;
            if (d.dbg_out) d.dbg_out[col + k] = out;
            dot += pw * widen<FP>(os);
          }
        }
      }
      dot = warp_sum(dot);
      if (lane == 0) {
        const uint32_t t = h[kRT], w = (gt >> 5);
        d.tile_red[8ull * t + w] = dot;
        d.tile_red[8ull * t + 4 + w] = FP(0);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);  // this warp no longer reads the tile region
    }
    if (pf) {
      atomicAdd(&L.prof[0], w_ready);
      atomicAdd(&L.prof[7], static_cast<unsigned long long>(clock64() - t_start));
    }
    return;
  }
  rc_setmaxnreg_dec56();
  if (warp == 8) {
    // ------------------------------------------------------------ producer
    // Tile regions are carved from the ring in tile order at their exact size
    // (wrapping to offset 0 when the tail does not fit); before a region is
    // written the producer waits, oldest first, for the in-flight tiles it
    // overlaps (and for the slot's previous tile).
    unsigned long long w_prod = 0, t_ring = 0, t_issue = 0;
    uint32_t i = 0;
    uint32_t head = 0;                   // next free byte
    uint32_t oldest = 0, inflight = 0;   // oldest in-flight tile (CTA-local index) and count
    uint32_t tail_off = 0;               // region start of the oldest in-flight tile
    for (uint32_t base = blockIdx.x; base < ntiles; base += 32u * gridDim.x) {
      const uint32_t my = base + lane * gridDim.x;
      uint4 m0 = make_uint4(0, 0, 0, 0), m1 = m0, m2 = m0;
      if (my < ntiles) {
        const uint4* r = reinterpret_cast<const uint4*>(d.tile_meta + static_cast<uint64_t>(kMCount) * my);
        m0 = r[0];
        m1 = r[1];
        m2 = r[2];
      }
      const uint32_t nb = min(32u, (ntiles - base + gridDim.x - 1) / gridDim.x);
      for (uint32_t k = 0; k < nb; ++k, ++i) {
        const long long tp0 = pf ? clock64() : 0;
        const uint32_t t = __shfl_sync(0xffffffffu, m0.x, k);
        const uint32_t ne = __shfl_sync(0xffffffffu, m0.z, k), pb = __shfl_sync(0xffffffffu, m0.w, k);
        const uint32_t npt = __shfl_sync(0xffffffffu, m1.x, k), cb = __shfl_sync(0xffffffffu, m1.y, k);
        const uint32_t ncam = __shfl_sync(0xffffffffu, m1.z, k);
        const uint64_t aux16 = __shfl_sync(0xffffffffu, m2.x, k), lin16 = __shfl_sync(0xffffffffu, m2.y, k);
        const AuxSec as = aux_sections(ne, npt);
        const RcLinSec ls = rc_lin_sections<FP>(ne, npt, ncam, HUBER);
        const Span s_p = span16(d.p + pcol0 + 3ull * pb, sizeof(SP) * 3ull * npt);
        const Span s_z = span16(d.z + pcol0 + 3ull * pb, sizeof(SP) * 3ull * npt);
        const uint32_t tcb = static_cast<uint32_t>(sizeof(FP) * kRcRec * ncam);
        const uint32_t o_aux = kRcHdrBytes, o_lin = o_aux + as.bytes, o_p = o_lin + ls.bytes;
        const uint32_t o_z = o_p + s_p.bytes, o_tc = o_z + s_z.bytes;
        const uint32_t o_v = o_tc + tcb;  // the preparer's v_p = D p (FP)
        const uint32_t o_x = o_v + r16(sizeof(FP) * 3ull * npt);  // x (when the deferred update is pending)
        const uint32_t sz = (o_x + (xpend ? s_p.bytes : 0u) + 127) / 128 * 128;
        // ---- room in the ring (warp-uniform bookkeeping)
        for (;;) {
          bool fits;
          if (inflight == 0) {
            if (head + sz > L.ring_bytes) head = 0;
            fits = true;
          } else if (inflight == kRcSlots) {
            fits = false;
          } else if (tail_off < head) {  // occupied [tail_off, head)
            if (head + sz <= L.ring_bytes) {
              fits = true;
            } else if (sz <= tail_off) {
              head = 0;
              fits = true;
            } else {
              fits = false;
            }
          } else {  // wrapped: free [head, tail_off)
            fits = head + sz <= tail_off;
          }
          if (fits) break;
          const uint32_t os = oldest % kRcSlots;
          mbar_wait_u(&empty[os], (oldest / kRcSlots) & 1u, bo, pf, w_prod);
          ++oldest;
          --inflight;
          tail_off = inflight ? slot_off[oldest % kRcSlots] : head;
        }
        const long long tp1 = pf ? clock64() : 0;
        const int s = static_cast<int>(i % kRcSlots);
        const uint32_t off = head;
        head += sz;
        if (inflight == 0) tail_off = off;
        ++inflight;
        unsigned char* rg = ring + off;
        if (lane == 0) {
          slot_off[s] = off;
          uint32_t* hh = reinterpret_cast<uint32_t*>(rg);
          hh[kRT] = t;
          hh[kRNe] = ne;
          hh[kRNpt] = npt;
          hh[kRNcam] = ncam;
          hh[kRPb] = pb;
          hh[kRCb] = cb;
          hh[kRDp] = s_p.delta;
          hh[kRDz] = s_z.delta;
          hh[kROAux] = o_aux;
          hh[kROLin] = o_lin;
          hh[kROP] = o_p;
          hh[kROZ] = o_z;
          hh[kROTc] = o_tc;
          hh[kROV] = o_v;
          hh[kROX] = o_x;
          // the tile's static + per-linearization blob: one bulk copy (contiguous, o_lin == o_aux + as.bytes)
          mbar_arrive_expect_tx(&blob[s], as.bytes + ls.bytes);
          bulk_g2s(rg + o_aux, d.tile_aux + 16 * aux16, as.bytes + ls.bytes, &blob[s]);
        }
        (void)lin16;
        if (pf) {
          const long long tp2 = clock64();
          t_ring += tp1 - tp0;
          t_issue += tp2 - tp1;
        }
      }
    }
    if (pf) {
      atomicAdd(&L.prof[2], w_prod);
      atomicAdd(&L.prof[4], t_ring);
      atomicAdd(&L.prof[5], t_issue);
    }
    return;
  }
  if (warp == 10) {
    // ------------------------------------------------------------ loader
    // p, z and the tile cameras' records of every tile: 16-byte cp.async by
    // every lane, completion counted on the tile's full barrier (small copies
    // stream faster through the LSU than as extra bulk copies)
    for (uint32_t i = 0; blockIdx.x + i * gridDim.x < ntiles; ++i) {
      const int s = static_cast<int>(i % kRcSlots);
      mbar_backoff_wait(&blob[s], (i / kRcSlots) & 1u, bo);  // header and blob (camera ids) are in place
      unsigned char* rg = ring + slot_off[s];
      const uint32_t* h = reinterpret_cast<const uint32_t*>(rg);
      const uint32_t ne = h[kRNe], npt = h[kRNpt], ncam = h[kRNcam], pb = h[kRPb];
      const uint32_t np16 = (h[kROZ] - h[kROP]) / 16, nz16 = dir ? np16 : 0u;
      constexpr uint32_t kRec16 = sizeof(FP) * kRcRec / 16;  // 16-byte chunks of one camera record
      const uint32_t nt16 = kRec16 * ncam;
      const char* psrc = reinterpret_cast<const char*>(d.p + pcol0 + 3ull * pb) - h[kRDp];
      const char* zsrc = reinterpret_cast<const char*>(d.z + pcol0 + 3ull * pb) - h[kRDz];
      const char* csrc = reinterpret_cast<const char*>(d.crec);
      // the tile's camera ids, from the aux blob once it has landed (the
      // producer's bulk copy): gathered straight from the per-camera records
      const uint32_t* tcam = reinterpret_cast<const uint32_t*>(rg + h[kROAux] + aux_sections(ne, npt).tcam);
      if (!(L.dbg & 32)) {
        for (uint32_t c = lane; c < np16; c += 32)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(rg + h[kROP] + 16 * c)),
                       "l"(psrc + 16 * c) : "memory");
        for (uint32_t c = lane; c < nz16; c += 32)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(rg + h[kROZ] + 16 * c)),
                       "l"(zsrc + 16 * c) : "memory");
        if (xpend) {  // x has the same column span (and alignment delta) as p
          const char* xsrc = reinterpret_cast<const char*>(d.xs + pcol0 + 3ull * pb) - h[kRDp];
          for (uint32_t c = lane; c < np16; c += 32)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(rg + h[kROX] + 16 * c)),
                         "l"(xsrc + 16 * c) : "memory");
        }
        for (uint32_t c = lane; c < nt16; c += 32)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(rg + h[kROTc] + 16 * c)),
                       "l"(csrc + sizeof(FP) * kRcRec * static_cast<uint64_t>(tcam[c / kRec16]) + 16 * (c % kRec16))
                       : "memory");
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_addr(&full[s])) : "memory");
    }
    return;
  }
  if (warp == 9) {
    // ------------------------------------------------------------ preparer
    // p <- z + beta p when the direction update is pending, v_p = D p into
    // the z slot (the consumers' gather source), then release the tile
    const FP beta = d.st->beta;
    unsigned long long w_full = 0;
    for (uint32_t i = 0; blockIdx.x + i * gridDim.x < ntiles; ++i) {
      const int s = static_cast<int>(i % kRcSlots);
      mbar_wait_u(&full[s], (i / kRcSlots) & 1u, bo, pf, w_full);
      mbar_backoff_wait(&blob[s], (i / kRcSlots) & 1u, bo);
      unsigned char* rg = ring + slot_off[s];
      const uint32_t* h = reinterpret_cast<const uint32_t*>(rg);
      const uint32_t npt = h[kRNpt];
      SP* pp = reinterpret_cast<SP*>(rg + h[kROP] + h[kRDp]);
      const SP* zz = reinterpret_cast<const SP*>(rg + h[kROZ] + h[kRDz]);
      FP* vv = reinterpret_cast<FP*>(rg + h[kROV]);
      const SP* xx = reinterpret_cast<const SP*>(rg + h[kROX] + h[kRDp]);
      const FP alpha = d.st->alpha;
      SP* xg = d.xs + pcol0 + 3ull * h[kRPb];
      const FP* DD = reinterpret_cast<const FP*>(rg + h[kROLin]);  // D at offset 0
      const uint32_t n3 = 3 * npt;
      constexpr int U = 4;
      for (uint32_t q0 = lane; q0 < n3; q0 += 32 * U) {
        SP pv[U], zv[U];
        FP dv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t q = q0 + 32 * u;
          if (q < n3) {
            pv[u] = pp[q];
            zv[u] = dir ? zz[q] : pv[u];
            dv[u] = DD[q];
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t q = q0 + 32 * u;
          if (q < n3) {
            if (xpend) xg[q] = pcg_x_value<FP, SP>(xx[q], pv[u], alpha);  // on p before the direction update
            const SP pn = dir ? pcg_dir_value<FP, SP>(zv[u], pv[u], beta) : pv[u];
            pp[q] = pn;
            vv[q] = dv[u] * widen<FP>(pn);  // == vt (k_pcg_dir)
          }
        }
      }
      mbar_arrive(&ready[s]);
    }
    if (pf) atomicAdd(&L.prof[3], w_full);
  }
}

// Per-camera HVP records (once per HVP): with the direction update pending
// (dir), p_c = z_c + beta p_c and v_c = D p_c first (k_pcg_dir_rest's camera
// half), plus the heavy tiles' point ranges. Record: M (row-major, M(i, k) =
// (Dw(e_k) v_w)_i), v_t, v_f, f v_k1, f v_k2.
template <typename FP, typename SP>
__global__ void k_rc_cams_pre(Dev<FP, SP> d, int dir, const uint64_t* rbeg, const uint64_t* rend, int nranges) {
  if (!d.st->iter_active || d.st->pcg_done) return;
  const FP beta = d.st->beta;
  const bool xpend = d.st->x_pending != 0;  // the last PCG update's x += alpha p (cameras, heavy-tile points)
  const FP alpha = d.st->alpha;
  if (dir && blockIdx.x == 0 && threadIdx.x == 0) d.st->dir_pending = 1;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const uint64_t t0 = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  for (uint64_t c = t0; c < d.nc; c += stride) {
    FP v[9], cam[9], pre[8];
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      const uint64_t col = 9 * c + k;
      if (xpend) d.xs[col] = pcg_x_value<FP, SP>(d.xs[col], d.p[col], alpha);
      if (dir) {
        const SP pi = pcg_dir_value<FP, SP>(d.z[col], d.p[col], beta);
        d.p[col] = pi;
        v[k] = d.D[col] * widen<FP>(pi);
        d.vt[col] = static_cast<arith_t<SP>>(v[k]);
      } else {
        v[k] = static_cast<FP>(d.vt[col]);
      }
      cam[k] = d.x[col];
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) pre[k] = d.cpre[static_cast<uint64_t>(kCamPre) * c + k];
    FP T[3][9];
    rot_basis<FP>(cam, pre, T);
    FP rec[kRcRec];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int k = 0; k < 3; ++k) rec[3 * i + k] = T[k][3 * i] * v[0] + T[k][3 * i + 1] * v[1] + T[k][3 * i + 2] * v[2];
    rec[9] = v[3];
    rec[10] = v[4];
    rec[11] = v[5];
    rec[12] = v[6];
    rec[13] = cam[6] * v[7];
    rec[14] = cam[6] * v[8];
    rec[15] = FP(0);
#pragma unroll
    for (int k = 0; k < kRcRec; ++k) d.crec[static_cast<uint64_t>(kRcRec) * c + k] = rec[k];
  }
  if (dir || xpend)
    for (int r = 0; r < nranges; ++r)
      for (uint64_t i = rbeg[r] + t0; i < rend[r]; i += stride) {
        if (xpend) d.xs[i] = pcg_x_value<FP, SP>(d.xs[i], d.p[i], alpha);
        if (!dir) continue;
        const SP pi = pcg_dir_value<FP, SP>(d.z[i], d.p[i], beta);
        d.p[i] = pi;
        d.vt[i] = static_cast<arith_t<SP>>(d.D[i] * widen<FP>(pi));
      }
}

// Camera side of the recompute HVP + p.Ap (pcg.hpp:332-340): 16 lanes per
// camera, lane v summing value v of the 15-value partials of the camera's tile
// copies (fixed tile-copy order, four rows in flight), then the 9 output lanes
// add the heavy tiles' 9-value partial slots and contract S with T_k =
// Dw(e_k) in closed form:
//   (sum_k,i T_k(i, j) S(k, i)) = w_j (-s tr S + s1 w.sigma + c2 w^T S w)
//                                 + s sigma_j + c ((S w)_j + (S^T w)_j),
// sigma = (S12 - S21, S20 - S02, S01 - S10), the chain coefficients s, c, s1,
// c2 of snavely.hpp:103-121. Phases as k_hvp_cams (0 fused, 1 per-rank sums
// -> red, 2 from red).
constexpr int kRcCamsPerBlock = 16;  // 16 lanes per camera (one per partial value), 256 threads

template <typename FP, typename SP>
__global__ void __launch_bounds__(16 * kRcCamsPerBlock) k_hvp_cams_rc(Dev<FP, SP> d, int phase) {
  if (!d.st->iter_active || d.st->pcg_done) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) d.st->x_pending = 0;  // applied by k_rc_cams_pre + k_hvp_rc
  __shared__ FP scratch[32];
  const int lane = threadIdx.x & 31, v = lane & 15, gbase = lane & 16;
  const uint32_t c = blockIdx.x * kRcCamsPerBlock + (threadIdx.x >> 4);
  const bool cam_ok = c < d.nc;
  FP out = FP(0);  // lane v < 9: value v of J_c^T q summed over the camera's edges
  if (phase != 2) {
    FP acc = FP(0);  // value v (15: padding) of the camera's tile copies, in tile-copy order
    if (cam_ok) {
      const uint32_t q1 = d.cam_tc_off[c + 1];
      uint32_t q = d.cam_tc_off[c];
      for (; q + 4 <= q1; q += 4) {  // four rows in flight
        FP r[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) r[u] = d.part15[static_cast<uint64_t>(kRcRec) * d.cam_tc_idx[q + u] + v];
#pragma unroll
        for (int u = 0; u < 4; ++u) acc += r[u];
      }
      for (; q < q1; ++q) acc += d.part15[static_cast<uint64_t>(kRcRec) * d.cam_tc_idx[q] + v];
    }
    FP S[kRcVals];
#pragma unroll
    for (int j = 0; j < kRcVals; ++j) S[j] = __shfl_sync(0xffffffffu, acc, gbase | j);
    if (cam_ok && v < 9) {
      const FP w0 = d.x[9ull * c], w1 = d.x[9ull * c + 1], w2 = d.x[9ull * c + 2], f = d.x[9ull * c + 6];
      const FP* pre = d.cpre + static_cast<uint64_t>(kCamPre) * c;
      const FP s = pre[4], cc = pre[5], s1 = pre[6], c2 = pre[7];
      if (v < 3) {
        const FP w[3] = {w0, w1, w2};
        const FP sig[3] = {S[5] - S[7], S[6] - S[2], S[1] - S[3]};  // S(k, i) at 3k + i
        FP Sw[3], STw[3];
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          Sw[j] = S[3 * j] * w0 + S[3 * j + 1] * w1 + S[3 * j + 2] * w2;
          STw[j] = S[j] * w0 + S[3 + j] * w1 + S[6 + j] * w2;
        }
        const FP wSw = w0 * Sw[0] + w1 * Sw[1] + w2 * Sw[2];
        const FP sc = -s * (S[0] + S[4] + S[8]) + s1 * (w0 * sig[0] + w1 * sig[1] + w2 * sig[2]) + c2 * wSw;
        FP o3[3];
#pragma unroll
        for (int j = 0; j < 3; ++j) o3[j] = w[j] * sc + s * sig[j] + cc * (Sw[j] + STw[j]);
        out = v == 0 ? o3[0] : (v == 1 ? o3[1] : o3[2]);
      } else if (v < 6) {
        out = v == 3 ? S[9] : (v == 4 ? S[10] : S[11]);
      } else {
        out = v == 6 ? S[12] : f * (v == 7 ? S[13] : S[14]);
      }
      if (d.n_heavy)  // heavy tiles: 9-value partial slots (k_hvp_tiles), flagged in camera-major order
        for (uint32_t q = d.cam_part_off[c]; q < d.cam_part_off[c + 1]; ++q)
          if (d.hflag[q]) out += d.part[9ull * q + v];
    }
  }
  FP mine = FP(0);
  if (phase == 1) {
    if (cam_ok && v < 9) d.red[9ull * c + v] = out;
  } else if (cam_ok && v < 9) {
    const bool freev = d.col_free[9ull * c];
    const uint64_t col = 9ull * c + v;
    const FP a = phase == 2 ? d.red[col] : out;
    const FP Dk = d.D[col];
    const FP damp = d.st->before_scaling ? d.st->lambda_solve * Dk * Dk : static_cast<FP>(d.st->lambda_solve);
    const FP pk = widen<FP>(d.p[col]);
    const FP o = freev ? damp * pk + Dk * a : FP(0);
    const SP os = narrow<SP>(o);
    d.ap[col] = os;
    if (d.dbg_out) d.dbg_out[col] = o;
    mine = pk * widen<FP>(os);
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

// Per-linearization lin blobs of the recompute path: point D, tile camera
// static records [R t f k1 k2 0] (R from camera_pre), Huber weights, point X.
template <typename FP, typename SP>
__global__ void k_tile_lin_rc(Dev<FP, SP> d, int force) {
  if (!force && !d.st->do_linearize) return;
  const uint32_t i = blockIdx.x;
  const uint32_t* m = d.tile_meta + static_cast<uint64_t>(kMCount) * i;
  const uint32_t eb = m[kMEb], ne = m[kMNe], pb = m[kMPb], npt = m[kMNpt], cb = m[kMCb], ncam = m[kMNcam];
  const uint32_t ne8 = (ne + kEdgePad - 1) / kEdgePad * kEdgePad;
  const RcLinSec ls = rc_lin_sections<FP>(ne, npt, ncam, d.w != nullptr);
  unsigned char* l = d.tile_lin + 16ull * m[kMLin16];
  FP* D = reinterpret_cast<FP*>(l + ls.D);
  for (uint32_t k = threadIdx.x; k < 3 * npt; k += blockDim.x) D[k] = d.D[9ull * d.nc + 3ull * pb + k];
  FP* cr = reinterpret_cast<FP*>(l + ls.cam);
  for (uint32_t k = threadIdx.x; k < kRcRec * ncam; k += blockDim.x) {
    const uint64_t c = d.tile_cams[cb + k / kRcRec];
    const uint32_t v = k % kRcRec;
    cr[k] = v < 9 ? d.cpre[static_cast<uint64_t>(kCamPre) * c + 8 + v] : (v < 15 ? d.x[9 * c + v - 6] : FP(0));
  }
  if (d.w) {
    FP* w = reinterpret_cast<FP*>(l + ls.w);
    for (uint32_t k = threadIdx.x; k < ne8; k += blockDim.x) w[k] = d.w[eb + k];
  }
  FP* X = reinterpret_cast<FP*>(l + ls.X);
  for (uint32_t k = threadIdx.x; k < 3 * npt; k += blockDim.x) X[k] = d.x[9ull * d.nc + 3ull * pb + k];
}

// hflag[q] = 1 for the camera-major partial slots of heavy tiles
template <typename FP, typename SP>
__global__ void k_mark_heavy_slots(Dev<FP, SP> d, uint8_t* hflag) {
  const uint32_t t = d.heavy_tiles[blockIdx.x];
  const uint32_t s0 = d.chunk_part_base[d.tile_chunk_base[t]], s1 = d.chunk_part_base[d.tile_chunk_base[t + 1]];
  for (uint32_t s = s0 + threadIdx.x; s < s1; s += blockDim.x) hflag[d.run_slot[s]] = 1;
}

// Full J (24 values per slot, SoA) recomputed by the linearize chain at x:
// the LinearSystem accessor surface when no Jacobian is stored.
template <typename FP, typename SP>
__global__ void k_eval_J(Dev<FP, SP> d, SP* out) {
  const uint32_t t = blockIdx.x;
  const uint32_t eb = d.tile_ebeg[t], ne = d.tile_ecnt[t], pb = d.tile_pbeg[t];
  const uint64_t pcol0 = 9ull * d.nc;
  for (uint32_t j = threadIdx.x; j < ne; j += blockDim.x) {
    const uint32_t e = eb + j;
    const uint32_t cam = d.d_cam[e];
    FP cp[9], X[3], jc[18], jp[6];
#pragma unroll
    for (int k = 0; k < 9; ++k) cp[k] = d.x[9ull * cam + k];
#pragma unroll
    for (int k = 0; k < 3; ++k) X[k] = d.x[pcol0 + 3ull * (pb + d.d_lpt[e]) + k];
    snavely_linearize<FP>(cp, X, FP(0), FP(0), nullptr, jc, jp, nullptr, d.cpre + static_cast<uint64_t>(kCamPre) * cam);
#pragma unroll
    for (int k = 0; k < 18; ++k) out[k * static_cast<uint64_t>(d.na) + e] = narrow<SP>(jc[k]);
#pragma unroll
    for (int k = 0; k < 6; ++k) out[(18 + k) * static_cast<uint64_t>(d.na) + e] = narrow<SP>(jp[k]);
  }
}

}  // namespace gb
