// Graph activation: everything the device needs that depends only on the
// graph structure (not on parameter values). Reference counterparts:
//   Graph::activate                  graph.hpp:59-83
//   VertexDescriptor::assign_columns vertex_descriptor.hpp:115-126
//   FactorDescriptor::activate       factor_descriptor.hpp:254-270
//   FactorDescriptor::build_incidence factor_descriptor.hpp:710-753
// The reference incidence CSRs are reproduced exactly (they are the
// bit-exact parity target) and then turned into the device layout described
// in DESIGN.md §Data layout: point tiles, camera-sorted edges inside each
// tile, warp-chunk camera runs and the camera -> partial-slot CSR.
#pragma once

#include <cstdint>
#include <vector>

namespace gb {

constexpr int kTileThreads = 256;  // CTA size of every tile kernel
constexpr int kTileEdges = 512;    // max edges of a normal tile (SMEM staging of the point side)
constexpr int kTilePoints = 256;   // max points of a tile
constexpr int kEdgePad = 8;        // tile edge ranges start on 8-edge boundaries (16-byte aligned rows)
constexpr int kJBlock = kTileEdges;  // tile slot ranges are padded to whole 512-slot blocks (J store blocks)
constexpr int kTileCams = 64;      // max distinct cameras of a normal tile (SMEM camera staging)
constexpr uint32_t kNoKey = 0xffffffffu;

struct Incidence {
  std::vector<uint64_t> vertex_of_segment;
  std::vector<uint64_t> offsets;
  std::vector<uint32_t> items;  // active factor index a; slot is implied (0 cams, 1 points)
};

struct ActivationInput {
  uint64_t nc = 0, np = 0, ne = 0;
  const uint32_t* cam = nullptr;
  const uint32_t* pt = nullptr;
  const uint8_t* level = nullptr;      // may be null (all 0)
  const uint8_t* cam_fixed = nullptr;  // may be null
  const uint8_t* pt_fixed = nullptr;   // may be null
  int active_level = 0;
  uint32_t tile_edge_cap = kTileEdges;  // greedy tile edge budget (<= kTileEdges; the recompute HVP uses less)
};

struct Activation {
  uint64_t nc = 0, np = 0, n_active = 0;
  int level = 0;
  std::vector<uint32_t> active;  // active factor a -> entry index (factor_descriptor.hpp:255-257)
  // reference column layout (free cameras first, then free points, insertion order)
  int64_t free_cams = 0, free_pts = 0, free_dims = 0;
  std::vector<int64_t> cam_col, pt_col;  // -1 when fixed (kFixedColumn)
  Incidence cam_inc, pt_inc;
  // internal point order: points sorted by (min active camera, id)
  std::vector<uint32_t> pt_order;  // internal i -> point id
  std::vector<uint32_t> pt_rank;   // point id -> internal i
  // tiles over internal points
  uint32_t ntiles = 0, nchunks = 0, nparts = 0;
  std::vector<uint32_t> tile_ebeg, tile_pbeg, tile_chunk_base;  // size ntiles+1; tile_ebeg padded
  std::vector<uint32_t> tile_ecnt;                              // real edges of each tile
  std::vector<uint32_t> normal_tiles, heavy_tiles;              // tile ids by kind
  uint64_t n_slots = 0;                                         // padded device edge slots (multiple of kJBlock)
  // device edge order d (tile-major, camera then factor index inside a tile),
  // padded: slots [tile_ebeg[t] + tile_ecnt[t], tile_ebeg[t+1]) are dummies
  std::vector<uint32_t> d_a;    // d -> active factor a (kNoKey for padding)
  std::vector<uint32_t> d_cam;  // d -> camera
  std::vector<uint16_t> d_lpt;  // d -> point index local to its tile
  std::vector<uint16_t> d_lcam; // d -> camera index local to its tile (normal tiles)
  std::vector<uint32_t> tile_cam_off, tile_cams;  // distinct cameras of each tile, ascending
  std::vector<uint32_t> pt_slot_off;  // internal point -> offsets into pt_slots (size np+1)
  std::vector<uint16_t> pt_slots;     // tile-local edge slots of each point, ascending
  // warp-chunk camera runs -> partial slots
  std::vector<uint32_t> chunk_part_base;  // size nchunks+1
  std::vector<uint32_t> cam_part_off;     // size nc+1
  std::vector<uint32_t> cam_part_idx;     // partial slots of each camera, ascending
};

// Throws std::invalid_argument on out-of-range indices.
void activate(const ActivationInput& in, Activation& out);

// Rank `rank` of `world`: a contiguous range of tiles balanced by edge slots,
// with its points and edges; cameras stay global (replicated). Incidence,
// columns and counts stay global. shard_range reports [tile0, tile1) and
// [point0, point1) in the full activation's internal order.
void shard_range(const Activation& full, int world, int rank, uint32_t* tile0, uint32_t* tile1, uint32_t* point0,
                 uint32_t* point1);
void shard(const Activation& full, int world, int rank, Activation& out);
// the same balance over raw tile arrays (tile_ebeg / tile_pbeg: ntiles + 1
// entries), shared by the host shard() and the per-rank device activation
void shard_bounds(const uint32_t* tile_ebeg, const uint32_t* tile_pbeg, uint32_t ntiles, int world, int rank,
                  uint32_t* tile0, uint32_t* tile1, uint32_t* point0, uint32_t* point1);

// building blocks shared with the device activation (activate_dev.cuh)
void greedy_tiles(const std::vector<uint32_t>& deg_int, std::vector<uint32_t>& tile_pbeg,
                  std::vector<uint32_t>& tile_ebeg, std::vector<uint32_t>& tile_of_pt, uint32_t edge_cap = kTileEdges);
// the same over a raw degree array; tile_of_pt may be null
void greedy_tiles(const uint32_t* deg_int, uint64_t np, std::vector<uint32_t>& tile_pbeg,
                  std::vector<uint32_t>& tile_ebeg, uint32_t* tile_of_pt, uint32_t edge_cap = kTileEdges);
void classify_tiles(Activation& out);
// FactorDescriptor::build_incidence for one slot (factor_descriptor.hpp:710-753)
void build_incidence_host(uint64_t nvert, const std::vector<uint32_t>& vert_of_a, const uint8_t* fixed, Incidence& inc);

}  // namespace gb
