// Bulk-copy pipelined HVP over normal tiles (LinearSystem::hvp,
// linear_system.hpp:104-115; hvp_forward factor_descriptor.hpp:372-407 and
// hvp_scatter :409-433).
//
// Same arithmetic, association order and outputs as k_hvp_tiles (so results
// are bit-identical), restructured for HBM bandwidth: one persistent CTA per
// SM, a producer warp and 16 consumer warps (one edge per consumer thread).
// The producer streams every byte a tile needs into a ring of shared-memory
// stages with 1-D bulk async copies (cp.async.bulk, completion counted on an
// mbarrier): the J rows (SoA, one contiguous run per row), local camera and
// point indices, Huber weights, the chunk partial-slot bases, the tile's
// point slot lists, and the tile's p, D and free masks. It also gathers the
// tile's cameras (D*p and, for the factored store, R and f) into the stage.
// Consumers therefore touch global memory only to write partial slots, ap
// and the per-warp dot partials, while the next stages' copies are in flight.
#pragma once

#include <algorithm>

#include "kernels.cuh"

namespace gb {

constexpr int kPipeConsumers = kTileEdges;          // one consumer thread per edge of a normal tile
constexpr int kPipeThreads = kPipeConsumers + 32;   // + one producer warp
constexpr int kPipeMaxStages = 4;

// byte offsets inside one stage (all 16-byte aligned)
struct PipeLayout {
  uint32_t hdr, J, lcam, lpt, w, cpb, camv, camr, pso, psl, p, D, cf;
  uint32_t stage_bytes, fixed_bytes, total_bytes;
  int stages, rows;
};

template <typename FP, typename SP>
inline PipeLayout pipe_layout(int rows, bool huber, uint32_t smem_budget) {
  using A = arith_t<SP>;
  PipeLayout L{};
  uint32_t o = 0;
  auto take = [&](uint64_t bytes) {
    const uint32_t r = o;
    o += static_cast<uint32_t>((bytes + 15) / 16 * 16);
    return r;
  };
  L.rows = rows;
  L.hdr = take(16 * 4);
  L.J = take(static_cast<uint64_t>(rows) * kTileEdges * sizeof(SP));
  L.lcam = take(kTileEdges * 2);
  L.lpt = take(kTileEdges * 2);
  L.w = huber ? take(kTileEdges * sizeof(FP)) : 0;
  L.cpb = take((kTileEdges / 32 + 1) * 4 + 32);
  L.camv = take(kTileCams * 9 * sizeof(A) + 32);
  L.camr = take(kTileCams * 10 * sizeof(FP) + 32);
  L.pso = take((kTilePoints + 1) * 4 + 32);
  L.psl = take(kTileEdges * 2 + 32);
  L.p = take(kTilePoints * 3 * sizeof(SP) + 32);
  L.D = take(kTilePoints * 3 * sizeof(FP) + 32);
  L.cf = take(kTilePoints * 3 + 32);
  L.stage_bytes = o;
  // after the stages: 2 mbarriers per stage, the point staging (kTileEdges x 3 A)
  L.fixed_bytes = 2 * kPipeMaxStages * 8 + static_cast<uint32_t>((kTileEdges * 3 * sizeof(A) + 15) / 16 * 16);
  const uint32_t avail = smem_budget > L.fixed_bytes ? smem_budget - L.fixed_bytes : 0;
  L.stages = static_cast<int>(std::min<uint32_t>(kPipeMaxStages, avail / L.stage_bytes));
  L.total_bytes = L.stages * L.stage_bytes + L.fixed_bytes;
  return L;
}

// ---- PTX helpers: mbarrier + 1-D bulk async copy global -> shared
__device__ inline uint32_t smem_addr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ inline void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ inline void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ inline void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile(
      "{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}" ::"r"(smem_addr(bar)),
      "r"(bytes)
      : "memory");
}
__device__ inline void mbar_arrive(uint64_t* bar) {
  asm volatile(
      "{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}" ::"r"(smem_addr(bar))
      : "memory");
}
__device__ inline void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred P;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      " @!P bra WAIT_%=;\n}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ inline void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
__device__ inline void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kPipeConsumers) : "memory"); }

// A byte range [src, src + bytes) widened to 16-byte granules: the copy
// source, its size, and where element 0 lands relative to the smem buffer.
struct Span {
  const char* src;
  uint32_t bytes, delta;
};
__device__ inline Span span16(const void* p, uint64_t bytes) {
  const uint64_t a = reinterpret_cast<uint64_t>(p);
  const uint64_t lo = a & ~uint64_t(15), hi = (a + bytes + 15) & ~uint64_t(15);
  return Span{reinterpret_cast<const char*>(lo), static_cast<uint32_t>(hi - lo), static_cast<uint32_t>(a - lo)};
}

enum PipeHdr : int { kHT = 0, kHNe, kHNpt, kHNcam, kHDcpb, kHDpso, kHDpsl, kHDp, kHDD, kHDcf, kHNe8, kHPb, kHDcv, kHDcr };

template <typename FP, typename SP>
__global__ void __launch_bounds__(kPipeThreads, 1) k_hvp_pipe(Dev<FP, SP> d, PipeLayout L) {
  using A = arith_t<SP>;
  if (!d.st->iter_active || d.st->pcg_done) return;
  extern __shared__ __align__(128) unsigned char pipe_smem[];
  const int S = L.stages;
  uint64_t* full = reinterpret_cast<uint64_t*>(pipe_smem + S * L.stage_bytes);
  uint64_t* empty = full + kPipeMaxStages;
  A* hstage = reinterpret_cast<A*>(empty + kPipeMaxStages);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);   // producer lane 0 (arrive + expect_tx)
      mbar_init(&empty[s], 1);  // consumer thread 0 after the tile's last barrier
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint64_t pcol0 = 9ull * d.nc;
  const uint32_t ntiles = d.n_normal;

  if (warp == kPipeConsumers / 32) {
    // ------------------------------------------------------------ producer
    // Tile records (tile_meta, 12 u32 each) are fetched 32 at a time, one per
    // lane, so the producer pays one dependent round trip per 32 tiles; every
    // other byte moves by bulk copy.
    uint32_t i = 0;
    for (uint32_t base = blockIdx.x; base < ntiles; base += 32u * gridDim.x) {
      const uint32_t my = base + lane * gridDim.x;
      uint4 m0 = make_uint4(0, 0, 0, 0), m1 = m0, m2 = m0;
      if (my < ntiles) {
        const uint4* r = reinterpret_cast<const uint4*>(d.tile_meta + 12ull * my);
        m0 = r[0];
        m1 = r[1];
        m2 = r[2];
      }
      const uint32_t nb = min(32u, (ntiles - base + gridDim.x - 1) / gridDim.x);
      for (uint32_t k = 0; k < nb; ++k, ++i) {
        const uint32_t t = __shfl_sync(0xffffffffu, m0.x, k), eb = __shfl_sync(0xffffffffu, m0.y, k);
        const uint32_t ne = __shfl_sync(0xffffffffu, m0.z, k), pb = __shfl_sync(0xffffffffu, m0.w, k);
        const uint32_t npt = __shfl_sync(0xffffffffu, m1.x, k), cb = __shfl_sync(0xffffffffu, m1.y, k);
        const uint32_t ncam = __shfl_sync(0xffffffffu, m1.z, k), ch0 = __shfl_sync(0xffffffffu, m1.w, k);
        const uint32_t ps0 = __shfl_sync(0xffffffffu, m2.x, k);
        const int s = static_cast<int>(i % S);
        if (i >= static_cast<uint32_t>(S)) mbar_wait(&empty[s], ((i / S) - 1) & 1);
        unsigned char* st = pipe_smem + s * L.stage_bytes;
        const uint32_t nch = (ne + 31) / 32;
        const uint32_t ne8 = (ne + kEdgePad - 1) / kEdgePad * kEdgePad;
        const uint64_t pc = pcol0 + 3ull * pb;
        const Span s_cpb = span16(d.chunk_part_base + ch0, 4ull * nch);
        const Span s_pso = span16(d.pt_slot_off + pb, 4ull * (npt + 1));
        const Span s_psl = span16(d.pt_slots + ps0, 2ull * ne);
        const Span s_p = span16(d.p + pc, sizeof(SP) * 3ull * npt);
        const Span s_D = span16(d.D + pc, sizeof(FP) * 3ull * npt);
        const Span s_cf = span16(d.col_free + pc, 3ull * npt);
        const Span s_cv = span16(d.tcv + 9ull * cb, sizeof(A) * 9ull * ncam);
        const Span s_cr = span16(d.tcr + 10ull * cb, sizeof(FP) * 10ull * ncam);
        const bool fact = d.jfact != 0;
        const uint32_t jrow = ne8 * static_cast<uint32_t>(sizeof(SP));
        const uint32_t total = L.rows * jrow + 2 * (ne8 * 2) +
                               (d.w ? ne8 * static_cast<uint32_t>(sizeof(FP)) : 0) + s_cpb.bytes + s_pso.bytes +
                               s_psl.bytes + s_p.bytes + s_D.bytes + s_cf.bytes + s_cv.bytes +
                               (fact ? s_cr.bytes : 0);
        if (lane == 0) {
          uint32_t* h = reinterpret_cast<uint32_t*>(st + L.hdr);
          h[kHT] = t;
          h[kHNe] = ne;
          h[kHNpt] = npt;
          h[kHNcam] = ncam;
          h[kHDcpb] = s_cpb.delta;
          h[kHDpso] = s_pso.delta;
          h[kHDpsl] = s_psl.delta;
          h[kHDp] = s_p.delta;
          h[kHDD] = s_D.delta;
          h[kHDcf] = s_cf.delta;
          h[kHNe8] = ne8;
          h[kHPb] = pb;
          h[kHDcv] = s_cv.delta;
          h[kHDcr] = s_cr.delta;
          mbar_arrive_expect_tx(&full[s], total);  // releases the header; completes when all bytes land
        }
        __syncwarp();
        // copies: J rows 0..rows-1, then lcam, lpt, cpb, pso, psl, p, D, cf, camera D*p, [R f], [w]
        const int nfixed = 9;
        const int ncopies = L.rows + nfixed + (fact ? 1 : 0) + (d.w ? 1 : 0);
        for (int q = lane; q < ncopies; q += 32) {
          if (q < L.rows) {
            bulk_g2s(st + L.J + static_cast<uint32_t>(q) * kTileEdges * sizeof(SP),
                     d.J + static_cast<uint64_t>(q) * d.na + eb, jrow, &full[s]);
            continue;
          }
          int c = q - L.rows;
          if (c >= nfixed && !fact) ++c;  // skip the R f copy
          switch (c) {
            case 0: bulk_g2s(st + L.lcam, d.d_lcam + eb, ne8 * 2, &full[s]); break;
            case 1: bulk_g2s(st + L.lpt, d.d_lpt + eb, ne8 * 2, &full[s]); break;
            case 2: bulk_g2s(st + L.cpb, s_cpb.src, s_cpb.bytes, &full[s]); break;
            case 3: bulk_g2s(st + L.pso, s_pso.src, s_pso.bytes, &full[s]); break;
            case 4: bulk_g2s(st + L.psl, s_psl.src, s_psl.bytes, &full[s]); break;
            case 5: bulk_g2s(st + L.p, s_p.src, s_p.bytes, &full[s]); break;
            case 6: bulk_g2s(st + L.D, s_D.src, s_D.bytes, &full[s]); break;
            case 7: bulk_g2s(st + L.cf, s_cf.src, s_cf.bytes, &full[s]); break;
            case 8: bulk_g2s(st + L.camv, s_cv.src, s_cv.bytes, &full[s]); break;
            case 9: bulk_g2s(st + L.camr, s_cr.src, s_cr.bytes, &full[s]); break;
            default: bulk_g2s(st + L.w, d.w + eb, ne8 * static_cast<uint32_t>(sizeof(FP)), &full[s]); break;
          }
        }
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const A lam = static_cast<A>(d.st->lambda_solve);
  const int before = d.st->before_scaling;
  const FP lam_fp = static_cast<FP>(d.st->lambda_solve);
  for (uint32_t i = 0;; ++i) {
    const uint32_t idx = blockIdx.x + i * gridDim.x;
    if (idx >= ntiles) break;
    const int s = static_cast<int>(i % S);
    mbar_wait(&full[s], (i / S) & 1);
    const unsigned char* st = pipe_smem + s * L.stage_bytes;
    const uint32_t* h = reinterpret_cast<const uint32_t*>(st + L.hdr);
    const uint32_t t = h[kHT], ne = h[kHNe], npt = h[kHNpt], pb = h[kHPb];
    const SP* sJ = reinterpret_cast<const SP*>(st + L.J);
    const uint16_t* slc = reinterpret_cast<const uint16_t*>(st + L.lcam);
    const uint16_t* slp = reinterpret_cast<const uint16_t*>(st + L.lpt);
    const uint32_t* scpb = reinterpret_cast<const uint32_t*>(st + L.cpb + h[kHDcpb]);
    const uint32_t* spso = reinterpret_cast<const uint32_t*>(st + L.pso + h[kHDpso]);
    const uint16_t* spsl = reinterpret_cast<const uint16_t*>(st + L.psl + h[kHDpsl]);
    const SP* sp = reinterpret_cast<const SP*>(st + L.p + h[kHDp]);
    const FP* sD = reinterpret_cast<const FP*>(st + L.D + h[kHDD]);
    const uint8_t* scf = st + L.cf + h[kHDcf];
    const A* camv = reinterpret_cast<const A*>(st + L.camv + h[kHDcv]);
    const FP* camr = reinterpret_cast<const FP*>(st + L.camr + h[kHDcr]);

    // ---- edge phase: thread j = edge j of the tile
    {
      const uint32_t j = tid;
      const bool valid = j < ne;
      const uint32_t jj = valid ? j : 0;
      const uint32_t lc = slc[jj], lp = slp[jj];
      A jc[18], jp[6];
      bool done = false;
      if constexpr (std::is_same<SP, FP>::value) {
        if (d.jfact) {
          FP U[6], R[9];
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            jc[k] = sJ[k * kTileEdges + jj];
            jc[9 + k] = sJ[(3 + k) * kTileEdges + jj];
          }
#pragma unroll
          for (int k = 0; k < 6; ++k) U[k] = sJ[(6 + k) * kTileEdges + jj];
          const FP dist = sJ[12 * kTileEdges + jj], n = sJ[13 * kTileEdges + jj];
          const FP p0 = sJ[14 * kTileEdges + jj], p1 = sJ[15 * kTileEdges + jj];
          const FP* rf = camr + 10 * lc;
#pragma unroll
          for (int k = 0; k < 9; ++k) R[k] = rf[k];
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            jc[3 + k] = U[k];
            jc[12 + k] = U[3 + k];
          }
          point_block<FP>(U, R, jp);
          intrinsic_cols<FP>(dist, n, p0, p1, rf[9], jc);
          done = true;
        }
      }
      if (!done) {
#pragma unroll
        for (int k = 0; k < 18; ++k) jc[k] = widen<A>(sJ[k * kTileEdges + jj]);
#pragma unroll
        for (int k = 0; k < 6; ++k) jp[k] = widen<A>(sJ[(18 + k) * kTileEdges + jj]);
      }
      const A wgt = d.w ? static_cast<A>(reinterpret_cast<const FP*>(st + L.w)[jj]) : A(1);
      const A* cv = camv + 9 * lc;
      A u0 = A(0), u1 = A(0), s0 = A(0), s1 = A(0);
#pragma unroll
      for (int k = 0; k < 9; ++k) {
        const A v = cv[k];
        u0 += jc[k] * v;
        u1 += jc[9 + k] * v;
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const A v = static_cast<A>(sD[3 * lp + k]) * widen<A>(sp[3 * lp + k]);  // == vt (k_pcg_dir)
        s0 += jp[k] * v;
        s1 += jp[3 + k] * v;
      }
      u0 += s0;
      u1 += s1;
      const A q0 = valid ? wgt * u0 : A(0), q1 = valid ? wgt * u1 : A(0);
      A g[9];
#pragma unroll
      for (int k = 0; k < 9; ++k) g[k] = jc[k] * q0 + jc[9 + k] * q1;
      {
        const uint32_t prev = __shfl_up_sync(0xffffffffu, lc, 1);
        const unsigned hm = __ballot_sync(0xffffffffu, valid && (lane == 0 || lc != prev));
        const unsigned vm = __ballot_sync(0xffffffffu, valid);
        run_reduce9_store<A, FP>(g, lane, hm, vm, hm ? scpb[warp] : 0u, d.part);
      }
      if (valid) {
#pragma unroll
        for (int k = 0; k < 3; ++k) hstage[j * 3 + k] = jp[k] * q0 + jp[3 + k] * q1;
      }
    }
    consumer_sync();

    // ---- point epilogue: warps 0..7, thread = point (same partition as k_hvp_tiles)
    if (tid < kTileThreads) {
      FP dot = FP(0);
      const uint32_t pi = tid;
      if (pi < npt) {
        A acc[3] = {A(0), A(0), A(0)};
        for (uint32_t q = spso[pi] - spso[0]; q < spso[pi + 1] - spso[0]; ++q) {
          const uint32_t sl = spsl[q];
#pragma unroll
          for (int k = 0; k < 3; ++k) acc[k] += hstage[sl * 3 + k];
        }
        const uint64_t col = pcol0 + 3ull * (pb + pi);
        const bool freev = scf[3 * pi];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const FP Dk = sD[3 * pi + k];
          const A damp = before ? static_cast<A>(lam_fp * Dk * Dk) : lam;
          const SP pk = sp[3 * pi + k];
          const A out = freev ? damp * widen<A>(pk) + static_cast<A>(Dk) * acc[k] : A(0);
          const SP o = narrow<SP>(out);
          d.ap[col + k] = o;
          if (d.dbg_out) d.dbg_out[col + k] = out;
          dot += widen<FP>(pk) * widen<FP>(o);
        }
      }
      dot = warp_sum(dot);
      if (lane == 0) d.tile_red[8ull * t + warp] = dot;
    }
    consumer_sync();
    if (tid == 0) mbar_arrive(&empty[s]);
  }
}

// Per-tile camera copies for the pipelined HVP: tcv[tile_cam_off[t] + lc] =
// vt of the tile's local camera lc (refreshed before every HVP), tcr = R, f
// (refreshed after every linearization, factored store only). They make each
// tile's camera data one contiguous bulk copy.
template <typename FP, typename SP>
__global__ void k_tcam_vt(Dev<FP, SP> d) {
  if (!d.st->iter_active || d.st->pcg_done) return;
  const uint64_t n = 9ull * d.ntcams;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    d.tcv[i] = d.vt[9ull * d.tile_cams[i / 9] + i % 9];
}
template <typename FP, typename SP>
__global__ void k_tcam_rf(Dev<FP, SP> d, int force) {
  if (!force && !d.st->do_linearize) return;
  const uint64_t n = 10ull * d.ntcams;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    d.tcr[i] = d.Rf[10ull * d.tile_cams[i / 10] + i % 10];
}

// Tile records for the pipelined HVP producer, in normal-tile list order:
// [t, ebeg, ecnt, pbeg, npt, cam_off, ncam, chunk_base, pt_slot_off[pbeg], 0, 0, 0]
template <typename FP, typename SP>
__global__ void k_tile_meta(Dev<FP, SP> d, uint32_t* meta) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < d.n_normal; i += gridDim.x * blockDim.x) {
    const uint32_t t = d.normal_tiles[i];
    uint32_t* m = meta + 12ull * i;
    m[0] = t;
    m[1] = d.tile_ebeg[t];
    m[2] = d.tile_ecnt[t];
    m[3] = d.tile_pbeg[t];
    m[4] = d.tile_pbeg[t + 1] - d.tile_pbeg[t];
    m[5] = d.tile_cam_off[t];
    m[6] = d.tile_cam_off[t + 1] - d.tile_cam_off[t];
    m[7] = d.tile_chunk_base[t];
    m[8] = d.pt_slot_off[d.tile_pbeg[t]];
    m[9] = m[10] = m[11] = 0;
  }
}

}  // namespace gb
