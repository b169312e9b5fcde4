// Linearize of the recompute path by run-aligned segments (k_lin_seg).
#pragma once

#include "hvp_rc.cuh"

namespace gb {

// Linearize of a normal tile on the recompute path (factor_descriptor.hpp:272-292,
// :322-370, unscaled half of :435-482): one thread per run-aligned segment of
// the aux blob (<= kSegSlots segments, one camera each). A thread runs its
// segment's edges in order and accumulates the run's 54 camera values (b, packed
// upper H) in registers, so the per-edge cost is the chain plus 54 FMAs instead
// of a cross-lane butterfly per (32-edge chunk, camera run). After the point
// epilogue the segment sums meet in shared memory (in the per-edge point
// buffer's space, 27 values at a time; segment rows of odd stride 27, so row
// writes and column reads are conflict-free) and are added per camera run in
// segment order into lpart[tile camera]; k_lin_cams sums a camera's entries in
// cam_tc order. Point b/H, D, chi^2 and the lin blob as k_lin_normal.
// 66 KB of shared memory and <= 168 registers: three CTAs per SM.
constexpr int kLinSegThreads = kSegSlots;
constexpr int kLinSegHalf = kLinVals / 2;  // values per shared-memory pass (and the odd row stride)
static_assert(kLinSegHalf * kSegSlots <= kTileEdges * 9, "segment sums fit the point buffer");
template <typename FP>
__host__ __device__ constexpr size_t lin_seg_smem() {
  return sizeof(FP) * (kTilePoints * 3 + kTileCams * 9 + kTileCams * kCamPre + kTileEdges * 9 + 32 + 2 * kTileEdges) +
         sizeof(uint16_t) * (2 * kTileEdges + kTilePoints + 8);
}

// camera value V of one edge folded into its accumulator, with jc and r
// pre-scaled by sqrt(w): b_V += j0V r0 + j1V r1, H(i, k) += j0i j0k + j1i j1k
// (two FMAs per value)
template <typename FP, int V>
__device__ __forceinline__ FP lin_seg_term(FP a, const FP* jc, FP r0, FP r1) {
  if constexpr (V < 9) {
    return fma(jc[V], r0, fma(jc[9 + V], r1, a));
  } else {
    constexpr int i = p9row(V - 9), k = p9col(V - 9);
    return fma(jc[i], jc[k], fma(jc[9 + i], jc[9 + k], a));
  }
}
template <typename FP, int... V>
__device__ __forceinline__ void lin_seg_acc(FP* acc, const FP* jc, FP r0, FP r1, std::integer_sequence<int, V...>) {
  ((acc[V] = lin_seg_term<FP, V>(acc[V], jc, r0, r1)), ...);
}

// element-wise async global -> shared copy (4 or 8 bytes; completion by cp_async_wait_all)
template <typename T>
__device__ __forceinline__ void cp_async_elem(T* dst, const T* src) {
  static_assert(sizeof(T) == 4 || sizeof(T) == 8, "cp.async.ca element size");
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(smem_addr(dst)), "l"(src), "n"(sizeof(T)) : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// HUB: Huber loss (d.w allocated); the squared-loss instantiation has no
// weight, sqrt or division in its edge loop (w = 1 folds away exactly).
template <typename FP, typename SP, bool HUB>
__global__ void __launch_bounds__(kLinSegThreads, 3) k_lin_seg(Dev<FP, SP> d, int force) {
  if (!force && !d.st->do_linearize) return;
  extern __shared__ __align__(16) unsigned char lin_smem[];
  FP* sX = reinterpret_cast<FP*>(lin_smem);
  FP* sC = sX + kTilePoints * 3;
  FP* sPre = sC + kTileCams * 9;
  FP* pst = sPre + kTileCams * kCamPre;
  FP* sA = pst;  // after the point epilogue
  FP* scratch = pst + kTileEdges * 9;
  FP* sObs = scratch + 32;  // [2][kTileEdges] the tile's observations
  uint16_t* sLpt = reinterpret_cast<uint16_t*>(sObs + 2 * kTileEdges);  // aux lpt, psl, pso
  uint16_t* sPsl = sLpt + kTileEdges;
  uint16_t* sPso = sPsl + kTileEdges;
  const int tid = threadIdx.x;
  const uint32_t i = blockIdx.x, t = d.normal_tiles[i];
  const uint32_t* m = d.tile_meta + static_cast<uint64_t>(kMCount) * i;
  const uint32_t eb = d.tile_ebeg[t], ne_t = d.tile_ecnt[t];
  const uint32_t pb = d.tile_pbeg[t], npt = d.tile_pbeg[t + 1] - pb;
  const uint32_t cb = d.tile_cam_off[t], ncam = d.tile_cam_off[t + 1] - cb;
  const uint64_t pcol0 = 9ull * d.nc;
  const AuxSec as = aux_sections(ne_t, npt);
  const unsigned char* aux = d.tile_aux + 16ull * m[kMAux16];
  const uint32_t sg = reinterpret_cast<const uint16_t*>(aux + as.seg)[tid];
  const uint32_t s0 = sg & 511u, cnt = sg >> 9;
  const uint32_t lc = cnt ? reinterpret_cast<const uint16_t*>(aux + as.lcam)[s0] : 0u;
  // prologue gathers as fire-and-forget async copies (one camera per thread),
  // so their latencies overlap instead of serializing loop iterations
  if (static_cast<uint32_t>(tid) < ncam) {
    const uint64_t c = d.tile_cams[cb + tid];
#pragma unroll
    for (int k = 0; k < 9; ++k) cp_async_elem(&sC[9 * tid + k], d.x + 9 * c + k);
#pragma unroll
    for (int k = 0; k < kCamPre; ++k) cp_async_elem(&sPre[kCamPre * tid + k], d.cpre + kCamPre * c + k);
  }
  for (uint32_t k = tid; k < npt * 3; k += blockDim.x) cp_async_elem(&sX[k], d.x + pcol0 + 3ull * pb + k);
  {  // observations and the aux index sections (16-byte aligned, 16-byte copies)
    const uint32_t ne8 = (ne_t + kEdgePad - 1) / kEdgePad * kEdgePad;
    constexpr uint32_t E16 = 16 / sizeof(FP);
    for (uint32_t k = tid; k < 2 * ne8 / E16; k += blockDim.x) {
      const uint32_t row = k / (ne8 / E16), c = k % (ne8 / E16);
      cp_async16(sObs + row * kTileEdges + c * E16, d.d_obs + static_cast<uint64_t>(row) * d.na + eb + c * E16);
    }
    for (uint32_t k = tid; k < ne8 / 8; k += blockDim.x) cp_async16(sLpt + 8 * k, aux + as.lpt + 16 * k);
    for (uint32_t k = tid; k < (ne_t + 7) / 8; k += blockDim.x) cp_async16(sPsl + 8 * k, aux + as.psl + 16 * k);
    for (uint32_t k = tid; k < (npt + 8) / 8; k += blockDim.x) cp_async16(sPso + 8 * k, aux + as.pso + 16 * k);
  }
  unsigned char* lb = d.tile_lin + 16ull * m[kMLin16];
  const RcLinSec lsec = rc_lin_sections<FP>(ne_t, npt, ncam, d.w != nullptr);
  cp_async_wait_all();
  __syncthreads();
  {
    FP* bx = reinterpret_cast<FP*>(lb + lsec.X);
    for (uint32_t k = tid; k < npt * 3; k += blockDim.x) bx[k] = sX[k];
    FP* bc = reinterpret_cast<FP*>(lb + lsec.cam);
    for (uint32_t k = tid; k < kRcRec * ncam; k += blockDim.x) {
      const uint32_t c = k / kRcRec, v = k % kRcRec;
      bc[k] = v < 9 ? sPre[kCamPre * c + 8 + v] : (v < 15 ? sC[9 * c + v - 6] : FP(0));
    }
  }
  FP acc[kLinVals];
#pragma unroll
  for (int v = 0; v < kLinVals; ++v) acc[v] = FP(0);
  FP chi = FP(0);
  FP* bw = reinterpret_cast<FP*>(lb + lsec.w);
  for (uint32_t k = 0; k < cnt; ++k) {
    const uint32_t j = s0 + k, e = eb + j;
    const uint32_t lp = sLpt[j];
    const FP o0 = sObs[j], o1 = sObs[kTileEdges + j];
    FP res[2], jc[18], jp[6];
    snavely_linearize<FP>(&sC[9 * lc], &sX[3 * lp], o0, o1, res, jc, jp, nullptr, &sPre[kCamPre * lc]);
    const FP s = res[0] * res[0] + res[1] * res[1];
    const FP w = HUB ? loss_weight<FP>(d.loss_kind, d.huber, s) : FP(1);
    chi += HUB ? loss_value<FP>(d.loss_kind, d.huber, s) : s;
    if (HUB) {
      d.w[e] = w;
      bw[j] = w;
    }
    const FP wr0 = w * res[0], wr1 = w * res[1];
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
    FP r0 = res[0], r1 = res[1];
    if (HUB) {  // robust loss: w J^T J = (sqrt(w) J)^T (sqrt(w) J), w J^T r = (sqrt(w) J)^T (sqrt(w) r)
      const FP sw = sqrt(w);
#pragma unroll
      for (int u = 0; u < 18; ++u) jc[u] *= sw;
      r0 *= sw;
      r1 *= sw;
    }
    lin_seg_acc<FP>(acc, jc, r0, r1, std::make_integer_sequence<int, kLinVals>{});
  }
  __syncthreads();  // pst complete

  // point epilogue (as k_lin_normal)
  FP gmax = FP(0);
  int fin = 1;
  for (uint32_t k = tid; k < npt; k += blockDim.x) {
    FP pa[9];
#pragma unroll
    for (int u = 0; u < 9; ++u) pa[u] = FP(0);
    for (uint32_t q = sPso[k]; q < sPso[k + 1]; ++q) {
      const uint32_t sl = sPsl[q];
#pragma unroll
      for (int u = 0; u < 9; ++u) pa[u] += pst[sl * 9 + u];
    }
    const uint64_t col = pcol0 + 3ull * (pb + k);
    const bool freev = d.col_free[col];
    const uint64_t pidx = static_cast<uint64_t>(pb + k);
#pragma unroll
    for (int u = 0; u < 3; ++u) {
      const FP bk = freev ? pa[u] : FP(0);
      d.b[col + u] = bk;
      const FP diag = freev ? pa[3 + p3(u, u)] : FP(0);
      const FP cl = clampv(diag, FP(d.st->clamp_min), FP(d.st->clamp_max));
      d.clamped[col + u] = freev ? cl : FP(0);
      const FP Dv = freev ? FP(1) / sqrt(cl) : FP(0);
      d.D[col + u] = Dv;
      reinterpret_cast<FP*>(lb + lsec.D)[3 * k + u] = Dv;
      if (freev) {
        fin &= (is_finite(bk) && is_finite(diag)) ? 1 : 0;
        gmax = fmax(gmax, fabs(bk));
      }
    }
#pragma unroll
    for (int u = 0; u < 6; ++u) d.Hp[6 * pidx + u] = freev ? pa[3 + u] : FP(0);
  }
  // camera runs: run c = segments [rseg[c], rseg[c + 1]), summed in segment order
  const uint16_t* rseg = reinterpret_cast<const uint16_t*>(aux + as.rseg);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    __syncthreads();  // pst / the previous half's reads done
#pragma unroll
    for (int v = 0; v < kLinSegHalf; ++v) sA[tid * kLinSegHalf + v] = acc[h * kLinSegHalf + v];
    __syncthreads();
    for (uint32_t it = tid; it < ncam * kLinSegHalf; it += blockDim.x) {
      const uint32_t c = it / kLinSegHalf, v = it % kLinSegHalf;
      FP a = FP(0);
      for (uint32_t q = rseg[c]; q < rseg[c + 1]; ++q) a += sA[q * kLinSegHalf + v];
      d.lpart[static_cast<uint64_t>(cb + c) * kLinVals + h * kLinSegHalf + v] = a;
    }
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

}  // namespace gb
