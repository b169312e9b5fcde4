// Device-side graph activation: the same structures as the
// host activate() (activate.cpp), bit for bit, built on the GPU with CUB radix
// sorts (stable) and scans. The only host step is the greedy tile partition
// over the internal-point degree array (one pass over np integers).
//
//   active edges        flags + exclusive scan + compaction (level <= L)
//   internal points     key = smallest active camera (atomicMin), stable sort
//   tiles               greedy_tiles() on the host over the degrees
//   device edge order   stable sort by (tile << 32 | camera) over factor order
//   camera runs / lcam  head flags + inclusive scans
//   partial-slot CSR    stable sort of run slots by camera + histogram scan
//   point slot lists    stable sort of (point rank, tile-local slot)
#pragma once

#include <cub/cub.cuh>

#include "activate.hpp"

namespace gb {
namespace actdev {

__global__ void k_flags(uint64_t ne, const uint32_t* cam, const uint32_t* pt, const uint8_t* level, int L,
                        uint32_t nc, uint32_t np, uint32_t* flag, int* bad) {
  for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < ne;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    if (cam[e] >= nc || pt[e] >= np) atomicOr(bad, 1);
    flag[e] = (!level || static_cast<int>(level[e]) <= L) ? 1u : 0u;
  }
}

__global__ void k_compact(uint64_t ne, const uint32_t* flag, const uint32_t* pos, const uint32_t* cam,
                          const uint32_t* pt, uint32_t* cam_a, uint32_t* pt_a, uint32_t* entry_a) {
  for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < ne;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    if (flag[e]) {
      const uint32_t a = pos[e];
      cam_a[a] = cam[e];
      pt_a[a] = pt[e];
      entry_a[a] = static_cast<uint32_t>(e);
    }
}

__global__ void k_fill_u32(uint64_t n, uint32_t v, uint32_t* out) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    out[i] = v;
}

__global__ void k_iota(uint64_t n, uint32_t* out) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    out[i] = static_cast<uint32_t>(i);
}

__global__ void k_point_stats(uint64_t na, const uint32_t* cam_a, const uint32_t* pt_a, uint32_t* key, uint32_t* deg) {
  for (uint64_t a = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; a < na;
       a += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    atomicMin(&key[pt_a[a]], cam_a[a]);
    atomicAdd(&deg[pt_a[a]], 1u);
  }
}

__global__ void k_rank(uint64_t np, const uint32_t* pt_order, const uint32_t* deg, uint32_t* pt_rank,
                       uint32_t* deg_int) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < np;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t p = pt_order[i];
    pt_rank[p] = static_cast<uint32_t>(i);
    deg_int[i] = deg[p];
  }
}

__device__ inline uint32_t tile_of_rank(const uint32_t* tile_pbeg, uint32_t ntiles, uint32_t r) {
  uint32_t lo = 0, hi = ntiles;  // last t with tile_pbeg[t] <= r, among non-empty tiles
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) / 2;
    if (tile_pbeg[mid] <= r) lo = mid; else hi = mid;
  }
  return lo;
}

// key (tile, camera) of every active edge; edges whose point lies outside this
// rank's internal range [p0, p1) get the sentinel tile ntiles (sorted last)
__global__ void k_edge_keys(uint64_t na, const uint32_t* cam_a, const uint32_t* pt_a, const uint32_t* pt_rank,
                            const uint32_t* tile_pbeg, uint32_t ntiles, uint32_t p0, uint32_t p1, uint64_t* key,
                            uint32_t* val) {
  for (uint64_t a = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; a < na;
       a += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t r = pt_rank[pt_a[a]];
    if (r < p0 || r >= p1) {
      key[a] = (static_cast<uint64_t>(ntiles) << 32) | 0xffffffffull;
    } else {
      const uint32_t t = tile_of_rank(tile_pbeg, ntiles, r - p0);
      key[a] = (static_cast<uint64_t>(t) << 32) | cam_a[a];
    }
    val[a] = static_cast<uint32_t>(a);
  }
}

// place edge k of the sorted order into its padded slot; emit head flags
template <typename FP>
__global__ void k_place(uint64_t na, const uint64_t* skey, const uint32_t* order, const uint32_t* cam_a,
                        const uint32_t* pt_a, const uint32_t* entry_a, const uint32_t* pt_rank, uint32_t p0,
                        const uint32_t* real_beg, const uint32_t* tile_ebeg, const uint32_t* tile_pbeg,
                        const double* obs, uint64_t ns, uint32_t* d_a, uint32_t* d_cam, uint16_t* d_lpt, FP* d_obs,
                        uint32_t* pkey, uint32_t* pval, uint32_t* head_cam, uint32_t* head_run) {
  for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < na;
       k += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t a = order[k];
    const uint32_t t = static_cast<uint32_t>(skey[k] >> 32);
    const uint32_t cam = static_cast<uint32_t>(skey[k]);
    const uint32_t j = static_cast<uint32_t>(k - real_beg[t]);
    const uint64_t d = tile_ebeg[t] + j;
    const uint32_t r = pt_rank[pt_a[a]] - p0;  // rank-local internal point
    d_a[d] = a;
    d_cam[d] = cam_a[a];
    d_lpt[d] = static_cast<uint16_t>(r - tile_pbeg[t]);
    const uint32_t e = entry_a[a];
    d_obs[d] = static_cast<FP>(obs[2ull * e]);
    d_obs[ns + d] = static_cast<FP>(obs[2ull * e + 1]);
    pkey[k] = r;
    pval[k] = j;
    const bool new_cam = j == 0 || static_cast<uint32_t>(skey[k - 1]) != cam;
    head_cam[k] = new_cam ? 1u : 0u;
    head_run[k] = (new_cam || (j & 31u) == 0) ? 1u : 0u;
  }
}

__global__ void k_tile_offsets(uint32_t ntiles, uint64_t na, const uint32_t* real_beg, const uint32_t* tile_ecnt,
                               const uint32_t* tile_chunk_base, const uint32_t* incl_cam, const uint32_t* incl_run,
                               uint32_t* tile_cam_off, uint32_t* chunk_part_base) {
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t <= ntiles; t += gridDim.x * blockDim.x) {
    if (t == ntiles) {
      tile_cam_off[t] = na ? incl_cam[na - 1] : 0;
      chunk_part_base[tile_chunk_base[t]] = na ? incl_run[na - 1] : 0;
      continue;
    }
    const uint32_t rb = real_beg[t];
    tile_cam_off[t] = rb ? incl_cam[rb - 1] : 0;
    const uint32_t nch = (tile_ecnt[t] + 31) / 32;
    for (uint32_t kk = 0; kk < nch; ++kk) {
      const uint32_t start = rb + 32 * kk;
      chunk_part_base[tile_chunk_base[t] + kk] = start ? incl_run[start - 1] : 0;
    }
  }
}

__global__ void k_runs(uint64_t na, const uint64_t* skey, const uint32_t* real_beg, const uint32_t* tile_ebeg,
                       const uint32_t* tile_cam_off, const uint32_t* head_cam, const uint32_t* incl_cam,
                       const uint32_t* head_run, const uint32_t* incl_run, uint16_t* d_lcam, uint32_t* tile_cams,
                       uint32_t* run_cam) {
  for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < na;
       k += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t t = static_cast<uint32_t>(skey[k] >> 32);
    const uint32_t cam = static_cast<uint32_t>(skey[k]);
    const uint64_t d = tile_ebeg[t] + (k - real_beg[t]);
    const uint32_t g = incl_cam[k] - 1;
    d_lcam[d] = static_cast<uint16_t>(min(g - tile_cam_off[t], 0xffffu));
    if (head_cam[k]) tile_cams[g] = cam;
    if (head_run[k]) run_cam[incl_run[k] - 1] = cam;
  }
}

// padding slots repeat the tile's last camera (and local camera index)
__global__ void k_pad(uint32_t ntiles, const uint32_t* tile_ebeg, const uint32_t* tile_ecnt, uint32_t* d_cam,
                      uint16_t* d_lcam) {
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < ntiles; t += gridDim.x * blockDim.x) {
    const uint32_t b = tile_ebeg[t], n = tile_ecnt[t];
    for (uint32_t d = b + n; d < tile_ebeg[t + 1]; ++d) {
      d_cam[d] = n ? d_cam[b + n - 1] : 0;
      d_lcam[d] = n ? d_lcam[b + n - 1] : 0;
    }
  }
}

__global__ void k_u32_to_u16(uint64_t n, const uint32_t* in, uint16_t* out) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    out[i] = static_cast<uint16_t>(in[i] & 0xffffu);
}

__global__ void k_hist(uint64_t n, const uint32_t* key, uint32_t* count) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    atomicAdd(&count[key[i]], 1u);
}

__global__ void k_col_free(uint32_t nc, uint32_t np, const uint8_t* cam_fixed, const uint8_t* pt_fixed,
                           const uint32_t* pt_order, uint8_t* col_free) {
  const uint64_t n = 9ull * nc + 3ull * np;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    bool f;
    if (i < 9ull * nc) f = !(cam_fixed && cam_fixed[i / 9]);
    else f = !(pt_fixed && pt_fixed[pt_order[(i - 9ull * nc) / 3]]);
    col_free[i] = f ? 1 : 0;
  }
}

// params: AoS user points <-> internal order
template <typename FP>
__global__ void k_gather_points(uint32_t np, const uint32_t* pt_order, const FP* user, FP* x_pts) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < 3ull * np;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    x_pts[i] = user[3ull * pt_order[i / 3] + i % 3];
}
template <typename FP>
__global__ void k_scatter_points(uint32_t np, const uint32_t* pt_order, const FP* x_pts, FP* user) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < 3ull * np;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    user[3ull * pt_order[i / 3] + i % 3] = x_pts[i];
}

inline int bits_for(uint64_t v) {
  int b = 1;
  while (b < 64 && (v >> b)) ++b;
  return b;
}

}  // namespace actdev
}  // namespace gb
