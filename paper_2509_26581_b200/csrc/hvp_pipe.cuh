// Bulk-copy pipelined HVP over normal tiles (LinearSystem::hvp,
// linear_system.hpp:104-115; hvp_forward factor_descriptor.hpp:372-407 and
// hvp_scatter :409-433).
//
// Same arithmetic and association order as k_hvp_tiles (results are
// bit-identical), restructured for HBM bandwidth: one persistent CTA per SM,
// a producer warp and 16 consumer warps (one edge per consumer thread). The
// producer streams every byte a tile needs into a ring of shared-memory
// stages with 1-D bulk async copies (cp.async.bulk, completion counted on an
// mbarrier). Small scattered copies are what limits a bulk-copy stream (a
// measured ~30-90 ns each, tools/tma_bench.cu), so a tile needs only
// rows + 4 copies: its J rows (SoA, one contiguous run per row), a static
// per-tile "aux" blob (edge camera/point indices, point slot lists, chunk
// partial-slot bases, free mask; built once per activation), a per-
// linearization "lin" blob (point D, camera R f, Huber weights), the tile's
// p (contiguous in the internal point order) and the tile's camera D*p copy
// (tcv, refreshed before each HVP). Consumers touch global memory only to
// write partial slots, ap and the per-warp dot partials.
#pragma once

#include <algorithm>

#include "kernels.cuh"

namespace gb {

constexpr int kPipeConsumers = kTileEdges;          // one consumer thread per edge of a normal tile
constexpr int kPipeThreads = kPipeConsumers + 64;   // + one producer (copy) warp + one preparer warp
constexpr int kPipeMaxStages = 4;

__host__ __device__ constexpr uint32_t r16(uint64_t b) { return static_cast<uint32_t>((b + 15) / 16 * 16); }

// per-camera record strides (elements) of the tile camera copies: 9 D*p values
// (tcv) and R, f (lin blob), padded to 16-byte records for vector loads
template <typename T>
__host__ __device__ constexpr int cam_stride() {
  return sizeof(T) == 8 ? 10 : 12;
}

// byte stride of one J row (and of one contribution row) in shared memory
template <typename T>
__host__ __device__ constexpr uint32_t pipe_jstride() {
  return static_cast<uint32_t>(jstore_stride<T>() * sizeof(T));  // == the J store block's row stride
}

// Section offsets inside a tile's aux blob (static) and lin blob (per
// linearization); identical on the host (sizes) and the device (reads).
// seg / rseg: the recompute HVP's run-aligned edge segments (hvp_rc.cuh):
// segment q = edges [start, start + count) of one camera run (start | count << 9),
// run lc = segments [rseg[lc], rseg[lc + 1])
constexpr int kSegSlots = 128;
struct AuxSec {
  uint32_t lcam, lpt, psl, pso, cf, seg, rseg, tcam, pos, bytes;
};
__host__ __device__ inline AuxSec aux_sections(uint32_t ne, uint32_t npt) {
  const uint32_t ne8 = (ne + kEdgePad - 1) / kEdgePad * kEdgePad;
  AuxSec a;
  a.lcam = 0;
  a.lpt = a.lcam + r16(2ull * ne8);
  a.psl = a.lpt + r16(2ull * ne8);
  a.pso = a.psl + r16(2ull * ne);
  a.cf = a.pso + r16(2ull * (npt + 1));
  a.seg = a.cf + r16(3ull * npt);
  a.rseg = a.seg + r16(2ull * kSegSlots);
  a.tcam = a.rseg + r16(2ull * (kTileCams + 1));  // the tile's cameras (global index), recompute HVP loader
  a.pos = a.tcam + r16(4ull * kTileCams);          // edge -> its position in the point-slot order (psl inverse)
  a.bytes = a.pos + r16(2ull * ne8);
  return a;
}
struct LinSec {
  uint32_t D, cr, w, bytes;
};
template <typename FP>
__host__ __device__ inline LinSec lin_sections(uint32_t ne, uint32_t npt, uint32_t ncam, bool fact, bool huber) {
  const uint32_t ne8 = (ne + kEdgePad - 1) / kEdgePad * kEdgePad;
  LinSec l;
  l.D = 0;
  l.cr = l.D + r16(sizeof(FP) * 3ull * npt);
  l.w = l.cr + (fact ? r16(sizeof(FP) * static_cast<uint64_t>(cam_stride<FP>()) * ncam) : 0u);
  l.bytes = l.w + (huber ? r16(sizeof(FP) * 1ull * ne8) : 0u);
  return l;
}

// byte offsets inside one stage (all 16-byte aligned)
struct PipeLayout {
  uint32_t hdr, J, aux, lin, p, z, camv, vt, gs, runs;
  uint32_t stage_bytes, fixed_bytes, total_bytes;
  int stages, rows;
  int dbg;  // experiments only (GB_PIPE_DBG): 1 skip camera reduction, 2 skip epilogue, 4 skip edge math,
            // 16 copy only the J rows
};

template <typename FP, typename SP>
inline PipeLayout pipe_layout(int rows, bool huber, bool fact, uint32_t smem_budget) {
  using A = arith_t<SP>;
  PipeLayout L{};
  uint32_t o = 0;
  auto take = [&](uint64_t bytes) {
    const uint32_t r = o;
    o += r16(bytes);
    return r;
  };
  L.rows = rows;
  L.hdr = take(32 * 4);
  // J rows at a padded stride (bank spread); rows 0..11 are reused for the
  // edges' camera (9) and point (3) contributions when sizeof(SP) == sizeof(A)
  L.J = take(static_cast<uint64_t>(rows) * pipe_jstride<SP>());
  L.aux = take(aux_sections(kTileEdges, kTilePoints).bytes);
  L.lin = take(lin_sections<FP>(kTileEdges, kTilePoints, kTileCams, fact, huber).bytes);
  L.p = take(kTilePoints * 3 * sizeof(SP) + 32);
  L.z = take(kTilePoints * 3 * sizeof(SP) + 32);
  L.camv = take(kTileCams * cam_stride<A>() * sizeof(A) + 32);
  L.vt = take(kTilePoints * 3 * sizeof(A));
  L.runs = take(8 * kTileEdges + 32);  // the tile's camera-run spans + storage slots (at most one run per edge)
  // camera / point contributions: over the J rows when SP and Arith have the
  // same width, else (bf16 storage) a 12-row area of the stage
  L.gs = sizeof(SP) == sizeof(A) ? L.J : take(12ull * pipe_jstride<A>());
  L.stage_bytes = o;
  // after the stages: 3 mbarriers per stage
  L.fixed_bytes = 3 * kPipeMaxStages * 8;
  const uint32_t avail = smem_budget > L.fixed_bytes ? smem_budget - L.fixed_bytes : 0;
  L.stages = static_cast<int>(std::min<uint32_t>(kPipeMaxStages, avail / L.stage_bytes));
  L.total_bytes = L.stages * L.stage_bytes + L.fixed_bytes;
  return L;
}


// N contiguous T from 16-byte aligned shared memory in 16-byte loads
template <typename T, int N>
__device__ inline void load16(const T* src, T (&out)[N]) {
  static_assert((N * sizeof(T)) % 16 == 0, "16-byte records");
  const uint4* s4 = reinterpret_cast<const uint4*>(src);
#pragma unroll
  for (int i = 0; i < static_cast<int>(N * sizeof(T) / 16); ++i) {
    const uint4 v = s4[i];
    memcpy(reinterpret_cast<char*>(out) + 16 * i, &v, 16);
  }
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

enum PipeHdr : int { kHT = 0, kHNe, kHNpt, kHNcam, kHDp, kHDcv, kHPb, kHDz, kHLpt, kHPsl, kHPso, kHDr, kHCf, kHCr, kHW, kHNr };

// stage index + parity of a ring of S stages (no integer division per tile)
struct RingPos {
  int s = 0;
  unsigned ph = 0;
  __device__ void next(int S) {
    if (++s == S) {
      s = 0;
      ph ^= 1u;
    }
  }
};

template <typename FP, typename SP>
__global__ void __launch_bounds__(kPipeThreads, 1) k_hvp_pipe(Dev<FP, SP> d, PipeLayout L) {
  using A = arith_t<SP>;
  if (!L.dbg && (!d.st->iter_active || d.st->pcg_done)) return;
  extern __shared__ __align__(128) unsigned char pipe_smem[];
  const int S = L.stages;
  uint64_t* full = reinterpret_cast<uint64_t*>(pipe_smem + S * L.stage_bytes);
  uint64_t* empty = full + kPipeMaxStages;
  uint64_t* ready = empty + kPipeMaxStages;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);   // producer lane 0 (arrive + expect_tx)
      mbar_init(&empty[s], kPipeConsumers / 32);  // every consumer warp, when done with the stage
      mbar_init(&ready[s], 32);  // every preparer lane, after preparing the tile's point values
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint64_t pcol0 = 9ull * d.nc;
  const uint32_t ntiles = d.n_normal;
  // p = z + beta p pending for this HVP's points (k_pcg_dir_rest did the rest)
  const bool dir = d.st->dir_pending != 0;
  const FP beta = d.st->beta;

  // Preparer warp: once a tile's bytes have landed, its points are prepared in
  // place: p <- z + beta p when the direction update is pending, and vt = D p
  // (the HVP's gather source), so consumers gather one value per point column
  // instead of three; then the tile is released to the consumers (ready).
  auto prepare = [&](const RingPos& rp) {
    const int sp_ = rp.s;
    mbar_wait(&full[sp_], rp.ph);
    unsigned char* st = pipe_smem + sp_ * L.stage_bytes;
    const uint32_t* h = reinterpret_cast<const uint32_t*>(st + L.hdr);
    const uint32_t npt = h[kHNpt];
    SP* pp = reinterpret_cast<SP*>(st + L.p + h[kHDp]);
    const SP* zz = reinterpret_cast<const SP*>(st + L.z + h[kHDz]);
    const FP* DD = reinterpret_cast<const FP*>(st + L.lin);  // lin section D at offset 0
    A* vv = reinterpret_cast<A*>(st + L.vt);
    const uint32_t n3 = 3 * npt;
    constexpr int U = 4;  // values per lane per pass, loads batched ahead of the stores
    for (uint32_t q0 = lane; q0 < n3; q0 += 32 * U) {
      SP pv[U], zv[U];
      FP dv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t q = q0 + 32 * u;
        if (q < n3) {  // lanes past the end read nothing (no cross-lane overlap with the stores)
          pv[u] = pp[q];
          zv[u] = dir ? zz[q] : pv[u];
          dv[u] = DD[q];
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t q = q0 + 32 * u;
        if (q < n3) {
          const SP pn = dir ? pcg_dir_value<FP, SP>(zv[u], pv[u], beta) : pv[u];
          pp[q] = pn;
          vv[q] = static_cast<A>(dv[u]) * widen<A>(pn);  // == vt (k_pcg_dir)
        }
      }
    }
    mbar_arrive(&ready[sp_]);  // every lane releases its own writes
  };
  if (warp == kPipeConsumers / 32) {
    // ------------------------------------------------------------ producer
    // Tile records (tile_meta, 12 u32 each) are fetched 32 at a time, one per
    // lane, so the producer pays one dependent round trip per 32 tiles; every
    // other byte moves by bulk copy.
    uint32_t i = 0;
    RingPos rp;
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
      for (uint32_t k = 0; k < nb; ++k, ++i, rp.next(S)) {
        const uint32_t t = __shfl_sync(0xffffffffu, m0.x, k), eb = __shfl_sync(0xffffffffu, m0.y, k);
        const uint32_t ne = __shfl_sync(0xffffffffu, m0.z, k), pb = __shfl_sync(0xffffffffu, m0.w, k);
        const uint32_t npt = __shfl_sync(0xffffffffu, m1.x, k), cb = __shfl_sync(0xffffffffu, m1.y, k);
        const uint32_t ncam = __shfl_sync(0xffffffffu, m1.z, k);
        const uint64_t aux16 = __shfl_sync(0xffffffffu, m2.x, k), lin16 = __shfl_sync(0xffffffffu, m2.y, k);
        const uint32_t slot0 = __shfl_sync(0xffffffffu, m2.z, k), nruns = __shfl_sync(0xffffffffu, m2.w, k);
        const int s = rp.s;
        if (i >= static_cast<uint32_t>(S)) mbar_wait(&empty[s], rp.ph ^ 1u);
        unsigned char* st = pipe_smem + s * L.stage_bytes;
        const AuxSec as = aux_sections(ne, npt);
        const LinSec ls = lin_sections<FP>(ne, npt, ncam, d.jfact != 0, d.w != nullptr);
        const Span s_p = span16(d.p + pcol0 + 3ull * pb, sizeof(SP) * 3ull * npt);
        const Span s_cv = span16(d.tcv + static_cast<uint64_t>(cam_stride<A>()) * cb,
                                 sizeof(A) * static_cast<uint64_t>(cam_stride<A>()) * ncam);
        const Span s_z = span16(d.z + pcol0 + 3ull * pb, sizeof(SP) * 3ull * npt);
        const Span s_r = span16(d.slot_span + slot0, 8ull * nruns);
        const bool small = !(L.dbg & 16);  // experiments: 16 = J rows only
        const uint32_t jblock = static_cast<uint32_t>(L.rows) * pipe_jstride<SP>();
        const uint32_t total =
            jblock +
            (small ? as.bytes + ls.bytes + s_p.bytes + s_cv.bytes + s_r.bytes + (dir ? s_z.bytes : 0u) : 0u);
        if (lane == 0) {
          uint32_t* h = reinterpret_cast<uint32_t*>(st + L.hdr);
          h[kHT] = t;
          h[kHNe] = ne;
          h[kHNpt] = npt;
          h[kHNcam] = ncam;
          h[kHDp] = s_p.delta;
          h[kHDcv] = s_cv.delta;
          h[kHPb] = pb;
          h[kHDz] = s_z.delta;
          h[kHLpt] = as.lpt;
          h[kHPsl] = as.psl;
          h[kHPso] = as.pso;
          h[kHDr] = s_r.delta;
          h[kHNr] = nruns;
          h[kHCf] = as.cf;
          h[kHCr] = ls.cr;
          h[kHW] = ls.w;
          mbar_arrive_expect_tx(&full[s], total);  // releases the header; completes when all bytes land
        }
        __syncwarp();
        const int ncopies = 1 + (small ? (dir ? 6 : 5) : 0);
        for (int q = lane; q < ncopies; q += 32) {
          switch (q) {
            case 0: bulk_g2s(st + L.J, d.J + jidx<SP>(eb, 0, L.rows), jblock, &full[s]); break;  // the tile's J block
            case 1: bulk_g2s(st + L.aux, d.tile_aux + 16 * aux16, as.bytes, &full[s]); break;
            case 2: bulk_g2s(st + L.lin, d.tile_lin + 16 * lin16, ls.bytes, &full[s]); break;
            case 3: bulk_g2s(st + L.p, s_p.src, s_p.bytes, &full[s]); break;
            case 4: bulk_g2s(st + L.camv, s_cv.src, s_cv.bytes, &full[s]); break;
            case 5: bulk_g2s(st + L.runs, s_r.src, s_r.bytes, &full[s]); break;
            default: bulk_g2s(st + L.z, s_z.src, s_z.bytes, &full[s]); break;
          }
        }
      }
    }
    return;
  }
  if (warp == kPipeConsumers / 32 + 1) {
    // ------------------------------------------------------------ preparer
    RingPos rp;
    for (uint32_t i = 0; blockIdx.x + i * gridDim.x < ntiles; ++i, rp.next(S)) prepare(rp);
    return;
  }

  // -------------------------------------------------------------- consumers
  const A lam = static_cast<A>(d.st->lambda_solve);
  const int before = d.st->before_scaling;
  const FP lam_fp = static_cast<FP>(d.st->lambda_solve);
  RingPos rp;
  for (uint32_t i = 0;; ++i, rp.next(S)) {
    const uint32_t idx = blockIdx.x + i * gridDim.x;
    if (idx >= ntiles) break;
    const int s = rp.s;
    mbar_wait(&ready[s], rp.ph);
    const unsigned char* st = pipe_smem + s * L.stage_bytes;
    const uint32_t* h = reinterpret_cast<const uint32_t*>(st + L.hdr);
    const uint32_t t = h[kHT], ne = h[kHNe], npt = h[kHNpt], pb = h[kHPb];
    const SP* sJ = reinterpret_cast<const SP*>(st + L.J);
    constexpr int JS = pipe_jstride<SP>() / sizeof(SP);  // J row stride (elements)
    constexpr int GS = pipe_jstride<A>() / sizeof(A);    // contribution row stride (elements)
    A* gs = reinterpret_cast<A*>(pipe_smem + s * L.stage_bytes + L.gs);  // per stage: the epilogue of
    // this tile may still read it while the other consumer half starts the next tile
    // section offsets of the aux / lin blobs, computed by the producer
    const unsigned char* aux = st + L.aux;
    const unsigned char* lin = st + L.lin;
    const uint16_t* slc = reinterpret_cast<const uint16_t*>(aux);
    const uint16_t* slp = reinterpret_cast<const uint16_t*>(aux + h[kHLpt]);
    const uint16_t* spsl = reinterpret_cast<const uint16_t*>(aux + h[kHPsl]);
    const uint16_t* spso = reinterpret_cast<const uint16_t*>(aux + h[kHPso]);
    const uint8_t* scf = aux + h[kHCf];
    const FP* sD = reinterpret_cast<const FP*>(lin);
    const FP* camr = reinterpret_cast<const FP*>(lin + h[kHCr]);
    const FP* sw = reinterpret_cast<const FP*>(lin + h[kHW]);
    const SP* sp = reinterpret_cast<const SP*>(st + L.p + h[kHDp]);
    const A* camv = reinterpret_cast<const A*>(st + L.camv + h[kHDcv]);
    const A* svt = reinterpret_cast<const A*>(st + L.vt);

    // ---- edge phase: thread j = edge j of the tile
    if (!(L.dbg & 4)) {
      const uint32_t j = tid;
      const bool valid = j < ne;
      const uint32_t jj = valid ? j : 0;  // indices of an invalid lane: edge 0's (its J column is its own)
      const uint32_t lc = slc[jj], lp = slp[jj];
      A jc[18], jp[6];
      bool done = false;
      if constexpr (std::is_same<SP, FP>::value) {
        if (d.jfact) {
          FP U[6], R[9];
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            jc[k] = sJ[k * JS + j];
            jc[9 + k] = sJ[(3 + k) * JS + j];
          }
#pragma unroll
          for (int k = 0; k < 6; ++k) U[k] = sJ[(6 + k) * JS + j];
          const FP dist = sJ[12 * JS + j], n = sJ[13 * JS + j];
          const FP p0 = sJ[14 * JS + j], p1 = sJ[15 * JS + j];
          FP rf[cam_stride<FP>()];
          load16<FP, cam_stride<FP>()>(camr + cam_stride<FP>() * lc, rf);
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
        for (int k = 0; k < 18; ++k) jc[k] = widen<A>(sJ[k * JS + j]);
#pragma unroll
        for (int k = 0; k < 6; ++k) jp[k] = widen<A>(sJ[(18 + k) * JS + j]);
      }
      const A wgt = d.w ? static_cast<A>(sw[jj]) : A(1);
      A cv[cam_stride<A>()];
      load16<A, cam_stride<A>()>(camv + cam_stride<A>() * lc, cv);
      A u0 = A(0), u1 = A(0), s0 = A(0), s1 = A(0);
#pragma unroll
      for (int k = 0; k < 9; ++k) {
        const A v = cv[k];
        u0 += jc[k] * v;
        u1 += jc[9 + k] * v;
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const A v = svt[3 * lp + k];
        s0 += jp[k] * v;
        s1 += jp[3 + k] * v;
      }
      u0 += s0;
      u1 += s1;
      const A q0 = valid ? wgt * u0 : A(0), q1 = valid ? wgt * u1 : A(0);
      A g[9];
#pragma unroll
      for (int k = 0; k < 9; ++k) g[k] = jc[k] * q0 + jc[9 + k] * q1;
      // contributions over this edge's own J column (thread j alone reads column j)
#pragma unroll
      for (int k = 0; k < 3; ++k) gs[(9 + k) * GS + j] = jp[k] * q0 + jp[3 + k] * q1;
      // camera contributions too: reduced per camera run after the sync
#pragma unroll
      for (int k = 0; k < 9; ++k) gs[k * GS + j] = g[k];
    }
    consumer_sync();

    // ---- point epilogue: one half of the consumers (alternating by tile), thread
    // = point, the same partition as k_hvp_tiles. The other half goes straight
    // on to the next tile's edge phase, so the epilogue overlaps it.
    const uint32_t half = i & 1;
    if ((static_cast<uint32_t>(tid) / kTileThreads) != half) {
      // ---- camera runs: the other half, one thread per (run, value), the
      // association order of chunk_runs_smem (identical to k_hvp_tiles)
      const uint32_t nr = h[kHNr];
      const uint2* spans = reinterpret_cast<const uint2*>(st + L.runs + h[kHDr]);
      for (uint32_t o = tid - (1 - half) * kTileThreads; o < 9 * nr && !(L.dbg & 1); o += kTileThreads) {
        const uint32_t r = o / 9, k = o - 9 * r;
        const uint2 sp2 = spans[r];
        const A* src = gs + k * GS;
        run_sum_store<A, FP>(src, sp2.x & 0xffffu, sp2.x >> 16, d.part + static_cast<uint64_t>(sp2.y) * 9 + k);
      }
    } else if (!(L.dbg & 2)) {
      FP dot = FP(0);
      const uint32_t pi = tid - half * kTileThreads;
      if (pi < npt) {
        A acc[3] = {A(0), A(0), A(0)};
        for (uint32_t q = spso[pi]; q < spso[pi + 1]; ++q) {
          const uint32_t sl = spsl[q];
#pragma unroll
          for (int k = 0; k < 3; ++k) acc[k] += gs[(9 + k) * GS + sl];
        }
        const uint64_t col = pcol0 + 3ull * (pb + pi);
        const bool freev = scf[3 * pi];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const FP Dk = sD[3 * pi + k];
          const A damp = before ? static_cast<A>(lam_fp * Dk * Dk) : lam;
          const SP pk = sp[3 * pi + k];  // direction update applied by the producer
          if (dir) d.p[col + k] = pk;
          const A out = freev ? damp * widen<A>(pk) + static_cast<A>(Dk) * acc[k] : A(0);
          const SP o = narrow<SP>(out);
          d.ap[col + k] = o;
          if (d.dbg_out) d.dbg_out[col + k] = out;
          dot += widen<FP>(pk) * widen<FP>(o);
        }
      }
      dot = warp_sum(dot);
      if (lane == 0) d.tile_red[8ull * t + (warp & 7)] = dot;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);  // this warp no longer reads stage s
  }
}

// Per-tile camera copies for the pipelined HVP: tcv[tile_cam_off[t] + lc] =
// vt of the tile's local camera lc, refreshed before every HVP, so each
// tile's camera data is one contiguous bulk copy.
template <typename FP, typename SP>
__global__ void k_tcam_vt(Dev<FP, SP> d) {
  if (!d.st->iter_active || d.st->pcg_done) return;
  constexpr int CS = cam_stride<arith_t<SP>>();
  const uint64_t n = static_cast<uint64_t>(CS) * d.ntcams;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t k = i % CS;
    d.tcv[i] = k < 9 ? d.vt[9ull * d.tile_cams[i / CS] + k] : arith_t<SP>(0);
  }
}
// Static per-tile aux blobs (once per activation): one CTA per normal tile.
template <typename FP, typename SP>
__global__ void k_tile_aux(Dev<FP, SP> d) {
  const uint32_t i = blockIdx.x;
  const uint32_t* m = d.tile_meta + static_cast<uint64_t>(kMCount) * i;
  const uint32_t eb = m[kMEb], ne = m[kMNe], pb = m[kMPb], npt = m[kMNpt], ch0 = m[kMCh0];
  const uint32_t ne8 = (ne + kEdgePad - 1) / kEdgePad * kEdgePad, nch = (ne + 31) / 32;
  const AuxSec as = aux_sections(ne, npt);
  unsigned char* a = d.tile_aux + 16ull * m[kMAux16];
  uint16_t* lcam = reinterpret_cast<uint16_t*>(a + as.lcam);
  uint16_t* lpt = reinterpret_cast<uint16_t*>(a + as.lpt);
  uint16_t* psl = reinterpret_cast<uint16_t*>(a + as.psl);
  uint16_t* pso = reinterpret_cast<uint16_t*>(a + as.pso);
  uint8_t* cf = a + as.cf;
  const uint32_t q0 = d.pt_slot_off[pb];
  for (uint32_t k = threadIdx.x; k < ne8; k += blockDim.x) {
    lcam[k] = d.d_lcam[eb + k];
    lpt[k] = d.d_lpt[eb + k];
  }
  uint16_t* pos = reinterpret_cast<uint16_t*>(a + as.pos);
  for (uint32_t k = threadIdx.x; k < ne; k += blockDim.x) {
    const uint16_t e = d.pt_slots[q0 + k];
    psl[k] = e;
    pos[e] = static_cast<uint16_t>(k);
  }
  for (uint32_t k = threadIdx.x; k <= npt; k += blockDim.x) pso[k] = static_cast<uint16_t>(d.pt_slot_off[pb + k] - q0);
  // camera-run slot spans: run r of chunk q (slot chunk_part_base[ch0 + q] + r)
  // covers tile edges [lo, hi), cut at chunk ends like the HVP tile kernels'
  if (threadIdx.x < 32) {
    const uint32_t lane = threadIdx.x;
    for (uint32_t q = 0; q < nch; ++q) {
      const uint32_t e = 32 * q + lane;
      const bool valid = e < ne;
      const uint32_t cam = valid ? d.d_lcam[eb + e] : 0u;
      const uint32_t prev = __shfl_up_sync(0xffffffffu, cam, 1);
      const unsigned heads = __ballot_sync(0xffffffffu, valid && (lane == 0 || cam != prev));
      if ((heads >> lane) & 1u) {
        const unsigned later = lane == 31 ? 0u : heads & (0xffffffffu << (lane + 1));
        const uint32_t hi = later ? 32 * q + __ffs(later) - 1 : min(32 * q + 32, ne);
        const uint32_t slot = d.chunk_part_base[ch0 + q] + __popc(heads & ((1u << lane) - 1u));
        d.slot_span[slot] = make_uint2(e | (hi << 16), d.run_slot[slot]);
      }
    }
    if (lane == 0) {
      uint32_t* mw = const_cast<uint32_t*>(m);
      mw[kMSlot0] = d.chunk_part_base[ch0];
      mw[kMNruns] = d.chunk_part_base[ch0 + nch] - d.chunk_part_base[ch0];
    }
  }
  for (uint32_t k = threadIdx.x; k < 3 * npt; k += blockDim.x) cf[k] = d.col_free[9ull * d.nc + 3ull * pb + k];
  // run-aligned segments of <= K edges, the smallest K >= 4 with at most
  // kSegSlots segments (each camera run is cut into ceil(len / K) pieces)
  __shared__ uint16_t run_lo[kTileCams + 1];
  const uint32_t ncam = m[kMNcam];
  {
    uint32_t* tcam = reinterpret_cast<uint32_t*>(a + as.tcam);
    for (uint32_t k = threadIdx.x; k < ncam; k += blockDim.x) tcam[k] = d.tile_cams[m[kMCb] + k];
  }
  for (uint32_t k = threadIdx.x; k < ne; k += blockDim.x) {
    const uint32_t lc = d.d_lcam[eb + k];
    if (k == 0 || d.d_lcam[eb + k - 1] != lc) run_lo[lc] = static_cast<uint16_t>(k);
  }
  if (threadIdx.x == 0) run_lo[ncam] = static_cast<uint16_t>(ne);
  __syncthreads();
  if (threadIdx.x == 0) {
    uint16_t* seg = reinterpret_cast<uint16_t*>(a + as.seg);
    uint16_t* rseg = reinterpret_cast<uint16_t*>(a + as.rseg);
    uint32_t K = 4;
    for (;; ++K) {
      uint32_t n = 0;
      for (uint32_t lc = 0; lc < ncam; ++lc) n += (run_lo[lc + 1] - run_lo[lc] + K - 1) / K;
      if (n <= kSegSlots) break;
    }
    uint32_t q = 0;
    for (uint32_t lc = 0; lc < ncam; ++lc) {
      rseg[lc] = static_cast<uint16_t>(q);
      for (uint32_t e = run_lo[lc]; e < run_lo[lc + 1]; e += K)
        seg[q++] = static_cast<uint16_t>(e | (min(K, run_lo[lc + 1] - e) << 9));
    }
    rseg[ncam] = static_cast<uint16_t>(q);
    for (; q < kSegSlots; ++q) seg[q] = 0;  // idle threads: count 0
  }
}

// Per-linearization lin blobs: point D, camera R f (factored store), Huber w.
template <typename FP, typename SP>
__global__ void k_tile_lin(Dev<FP, SP> d, int force) {
  if (!force && !d.st->do_linearize) return;
  const uint32_t i = blockIdx.x;
  const uint32_t* m = d.tile_meta + static_cast<uint64_t>(kMCount) * i;
  const uint32_t eb = m[kMEb], ne = m[kMNe], pb = m[kMPb], npt = m[kMNpt], cb = m[kMCb], ncam = m[kMNcam];
  const uint32_t ne8 = (ne + kEdgePad - 1) / kEdgePad * kEdgePad;
  const LinSec ls = lin_sections<FP>(ne, npt, ncam, d.jfact != 0, d.w != nullptr);
  unsigned char* l = d.tile_lin + 16ull * m[kMLin16];
  FP* D = reinterpret_cast<FP*>(l + ls.D);
  for (uint32_t k = threadIdx.x; k < 3 * npt; k += blockDim.x) D[k] = d.D[9ull * d.nc + 3ull * pb + k];
  if (d.jfact) {
    FP* cr = reinterpret_cast<FP*>(l + ls.cr);
    constexpr int CS = cam_stride<FP>();
    for (uint32_t k = threadIdx.x; k < CS * ncam; k += blockDim.x)
      cr[k] = k % CS < 10 ? d.Rf[10ull * d.tile_cams[cb + k / CS] + k % CS] : FP(0);
  }
  if (d.w) {
    FP* w = reinterpret_cast<FP*>(l + ls.w);
    for (uint32_t k = threadIdx.x; k < ne8; k += blockDim.x) w[k] = d.w[eb + k];
  }
}

}  // namespace gb
