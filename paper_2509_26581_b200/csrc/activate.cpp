#include "activate.hpp"

#include <algorithm>
#include <stdexcept>
#include <string>

namespace gb {

namespace {

// Counting sort of `items` (already in ascending order of the secondary key)
// by a dense primary key: a stable CSR build.
void stable_bucket(const std::vector<uint32_t>& key, uint64_t nkeys, const std::vector<uint32_t>& items,
                   std::vector<uint64_t>& off, std::vector<uint32_t>& sorted) {
  off.assign(nkeys + 1, 0);
  for (uint32_t it : items) ++off[key[it] + 1];
  for (uint64_t k = 0; k < nkeys; ++k) off[k + 1] += off[k];
  std::vector<uint64_t> cur(off.begin(), off.end() - 1);
  sorted.resize(items.size());
  for (uint32_t it : items) sorted[cur[key[it]]++] = it;
}

// FactorDescriptor::build_incidence (factor_descriptor.hpp:710-753) for one
// slot: segments over free vertices with >= 1 active factor, ascending vertex;
// items in ascending active-factor order.
void build_incidence(uint64_t nvert, const std::vector<uint32_t>& vert_of_a, const uint8_t* fixed,
                     Incidence& inc) {
  const uint64_t na = vert_of_a.size();
  std::vector<uint64_t> counts(nvert, 0);
  for (uint64_t a = 0; a < na; ++a) {
    const uint32_t v = vert_of_a[a];
    if (!(fixed && fixed[v])) ++counts[v];
  }
  inc.vertex_of_segment.clear();
  std::vector<uint64_t> seg_of(nvert, UINT64_MAX);
  for (uint64_t v = 0; v < nvert; ++v)
    if (counts[v]) {
      seg_of[v] = inc.vertex_of_segment.size();
      inc.vertex_of_segment.push_back(v);
    }
  inc.offsets.assign(inc.vertex_of_segment.size() + 1, 0);
  for (uint64_t s = 0; s < inc.vertex_of_segment.size(); ++s)
    inc.offsets[s + 1] = inc.offsets[s] + counts[inc.vertex_of_segment[s]];
  inc.items.resize(inc.offsets.back());
  std::vector<uint64_t> cur(inc.offsets.begin(), inc.offsets.end() - 1);
  for (uint64_t a = 0; a < na; ++a) {
    const uint32_t v = vert_of_a[a];
    if (fixed && fixed[v]) continue;
    inc.items[cur[seg_of[v]]++] = static_cast<uint32_t>(a);
  }
}


// Greedy tile partition over internal-point degrees (shared by the host and
// the device activation): <= kTileEdges edges and <= kTilePoints points per
// tile; a point with more than kTileEdges edges is a tile of its own.
// tile_ebeg here is the UNPADDED edge prefix.
}  // namespace

void greedy_tiles(const std::vector<uint32_t>& deg_int, std::vector<uint32_t>& tile_pbeg,
                  std::vector<uint32_t>& tile_ebeg, std::vector<uint32_t>& tile_of_pt, uint32_t edge_cap) {
  tile_of_pt.resize(deg_int.size());
  greedy_tiles(deg_int.data(), deg_int.size(), tile_pbeg, tile_ebeg, tile_of_pt.data(), edge_cap);
}

void greedy_tiles(const uint32_t* deg_int, uint64_t np, std::vector<uint32_t>& tile_pbeg,
                  std::vector<uint32_t>& tile_ebeg, uint32_t* tile_of_pt, uint32_t edge_cap) {
  const uint64_t cap = std::min<uint64_t>(edge_cap, kTileEdges);
  tile_pbeg.assign(1, 0);
  tile_ebeg.assign(1, 0);
  tile_pbeg.reserve(np / 64 + 2);
  tile_ebeg.reserve(np / 64 + 2);
  uint64_t te = 0, tp = 0, ecount = 0;
  for (uint64_t i = 0; i < np; ++i) {
    const uint64_t d = deg_int[i];
    const bool heavy = d > static_cast<uint64_t>(kTileEdges);
    if (tp > 0 && (heavy || te + d > cap || tp >= static_cast<uint64_t>(kTilePoints))) {
      tile_pbeg.push_back(static_cast<uint32_t>(i));
      tile_ebeg.push_back(static_cast<uint32_t>(ecount));
      te = tp = 0;
    }
    if (tile_of_pt) tile_of_pt[i] = static_cast<uint32_t>(tile_pbeg.size() - 1);
    te += d;
    tp += 1;
    ecount += d;
    if (heavy) {
      tile_pbeg.push_back(static_cast<uint32_t>(i + 1));
      tile_ebeg.push_back(static_cast<uint32_t>(ecount));
      te = tp = 0;
    }
  }
  if (tp > 0 || tile_pbeg.size() == 1) {
    tile_pbeg.push_back(static_cast<uint32_t>(np));
    tile_ebeg.push_back(static_cast<uint32_t>(ecount));
  }
}

// normal tiles: <= kTileEdges edges and <= kTileCams distinct cameras (the
// shared-memory kernels); everything else goes through the generic kernels
void classify_tiles(Activation& out) {
  out.normal_tiles.clear();
  out.heavy_tiles.clear();
  for (uint32_t t = 0; t < out.ntiles; ++t) {
    const bool heavy = out.tile_ecnt[t] > static_cast<uint32_t>(kTileEdges) ||
                       out.tile_cam_off[t + 1] - out.tile_cam_off[t] > static_cast<uint32_t>(kTileCams);
    (heavy ? out.heavy_tiles : out.normal_tiles).push_back(t);
  }
}

namespace {

// warp chunks (32 real edges from the tile start), their camera runs and the
// camera -> partial-slot CSR (slot order)
void build_partial_plan(Activation& out) {
  out.tile_chunk_base.assign(out.ntiles + 1, 0);
  for (uint32_t t = 0; t < out.ntiles; ++t)
    out.tile_chunk_base[t + 1] = out.tile_chunk_base[t] + (out.tile_ecnt[t] + 31) / 32;
  out.nchunks = out.tile_chunk_base[out.ntiles];
  out.chunk_part_base.assign(out.nchunks + 1, 0);
  std::vector<uint32_t> run_cam;
  for (uint32_t t = 0; t < out.ntiles; ++t) {
    const uint32_t eb = out.tile_ebeg[t], ee = eb + out.tile_ecnt[t];
    for (uint32_t k = 0; k < (out.tile_ecnt[t] + 31) / 32; ++k) {
      const uint32_t ch = out.tile_chunk_base[t] + k;
      uint32_t runs = 0;
      for (uint32_t d = eb + 32 * k; d < std::min(ee, eb + 32 * k + 32); ++d)
        if (d == eb + 32 * k || out.d_cam[d] != out.d_cam[d - 1]) {
          ++runs;
          run_cam.push_back(out.d_cam[d]);
        }
      out.chunk_part_base[ch + 1] = out.chunk_part_base[ch] + runs;
    }
  }
  out.nparts = out.chunk_part_base[out.nchunks];
  std::vector<uint32_t> slots(out.nparts);
  for (uint32_t s2 = 0; s2 < out.nparts; ++s2) slots[s2] = s2;
  std::vector<uint64_t> off;
  stable_bucket(run_cam, out.nc, slots, off, out.cam_part_idx);
  out.cam_part_off.assign(out.nc + 1, 0);
  for (uint64_t c = 0; c <= out.nc; ++c) out.cam_part_off[c] = static_cast<uint32_t>(off[c]);
}

}  // namespace

void activate(const ActivationInput& in, Activation& out) {
  out = Activation();
  out.nc = in.nc;
  out.np = in.np;
  out.level = in.active_level;
  for (uint64_t i = 0; i < in.ne; ++i) {
    if (in.cam[i] >= in.nc)
      throw std::invalid_argument("add_factor: slot 0 references unknown vertex id " + std::to_string(in.cam[i]));
    if (in.pt[i] >= in.np)
      throw std::invalid_argument("add_factor: slot 1 references unknown vertex id " + std::to_string(in.pt[i]));
  }

  // active list (factor_descriptor.hpp:255-257)
  out.active.reserve(in.ne);
  for (uint64_t i = 0; i < in.ne; ++i)
    if (!in.level || static_cast<int>(in.level[i]) <= in.active_level) out.active.push_back(static_cast<uint32_t>(i));
  const uint64_t na = out.n_active = out.active.size();

  // columns (vertex_descriptor.hpp:115-126, graph.hpp:70-71): cameras then points
  int64_t next = 0;
  out.cam_col.assign(in.nc, -1);
  for (uint64_t c = 0; c < in.nc; ++c)
    if (!(in.cam_fixed && in.cam_fixed[c])) {
      out.cam_col[c] = next;
      next += 9;
      ++out.free_cams;
    }
  out.pt_col.assign(in.np, -1);
  for (uint64_t p = 0; p < in.np; ++p)
    if (!(in.pt_fixed && in.pt_fixed[p])) {
      out.pt_col[p] = next;
      next += 3;
      ++out.free_pts;
    }
  out.free_dims = next;

  std::vector<uint32_t> cam_of_a(na), pt_of_a(na);
  for (uint64_t a = 0; a < na; ++a) {
    cam_of_a[a] = in.cam[out.active[a]];
    pt_of_a[a] = in.pt[out.active[a]];
  }
  build_incidence(in.nc, cam_of_a, in.cam_fixed, out.cam_inc);
  build_incidence(in.np, pt_of_a, in.pt_fixed, out.pt_inc);

  // internal point order: stable bucket of points by their smallest active
  // camera (points sharing camera sets become neighbours -> tiles touch few
  // cameras); points without active edges go last.
  std::vector<uint32_t> key(in.np, kNoKey);
  std::vector<uint32_t> deg(in.np, 0);
  for (uint64_t a = 0; a < na; ++a) {
    const uint32_t p = pt_of_a[a];
    key[p] = std::min(key[p], cam_of_a[a]);
    ++deg[p];
  }
  {
    std::vector<uint32_t> k2(in.np), ids(in.np);
    for (uint64_t p = 0; p < in.np; ++p) {
      k2[p] = key[p] == kNoKey ? static_cast<uint32_t>(in.nc) : key[p];
      ids[p] = static_cast<uint32_t>(p);
    }
    std::vector<uint64_t> off;
    stable_bucket(k2, in.nc + 1, ids, off, out.pt_order);
  }
  out.pt_rank.assign(in.np, 0);
  for (uint64_t i = 0; i < in.np; ++i) out.pt_rank[out.pt_order[i]] = static_cast<uint32_t>(i);

  // tiles: greedy over internal points, <= kTileEdges edges and <= kTilePoints
  // points; a point with more than kTileEdges edges is a tile of its own
  // ("heavy" tile, processed chunk by chunk). Only degrees are needed, so the
  // device activation runs the same loop on the host over the degree array.
  std::vector<uint32_t> deg_int(in.np);
  for (uint64_t i = 0; i < in.np; ++i) deg_int[i] = deg[out.pt_order[i]];
  std::vector<uint32_t> tile_of_pt;
  greedy_tiles(deg_int, out.tile_pbeg, out.tile_ebeg, tile_of_pt, in.tile_edge_cap);
  out.ntiles = static_cast<uint32_t>(out.tile_pbeg.size() - 1);

  // device edge order: active edges sorted by camera (stable in a), then
  // stably bucketed by tile -> inside a tile: (camera, a). Tiles start on
  // kJBlock boundaries (one J store block per normal tile); the padding slots
  // are dummies.
  std::vector<uint32_t> order;
  {
    std::vector<uint32_t> all(na);
    for (uint64_t a = 0; a < na; ++a) all[a] = static_cast<uint32_t>(a);
    std::vector<uint64_t> off;
    std::vector<uint32_t> by_cam;
    stable_bucket(cam_of_a, in.nc, all, off, by_cam);
    std::vector<uint32_t> tile_of_a(na);
    for (uint64_t a = 0; a < na; ++a) tile_of_a[a] = tile_of_pt[out.pt_rank[pt_of_a[a]]];
    stable_bucket(tile_of_a, out.ntiles, by_cam, off, order);
  }
  out.tile_ecnt.resize(out.ntiles);
  std::vector<uint32_t> real_beg(out.tile_ebeg);  // unpadded prefix (built above)
  uint64_t slot = 0;
  for (uint32_t t = 0; t < out.ntiles; ++t) {
    out.tile_ecnt[t] = real_beg[t + 1] - real_beg[t];
    out.tile_ebeg[t] = static_cast<uint32_t>(slot);
    slot += (out.tile_ecnt[t] + kJBlock - 1) / kJBlock * kJBlock;
  }
  if (slot > 0xffffffffull) throw std::invalid_argument("more than 2^32 padded edge slots");
  out.tile_ebeg[out.ntiles] = static_cast<uint32_t>(slot);
  out.n_slots = slot;
  out.d_a.assign(slot, kNoKey);
  out.d_cam.assign(slot, 0);
  out.d_lpt.assign(slot, 0);
  for (uint32_t t = 0; t < out.ntiles; ++t) {
    for (uint32_t j = 0; j < out.tile_ecnt[t]; ++j) {
      const uint32_t a = order[real_beg[t] + j];
      const uint32_t d = out.tile_ebeg[t] + j;
      const uint32_t r = out.pt_rank[pt_of_a[a]];
      out.d_a[d] = a;
      out.d_cam[d] = cam_of_a[a];
      out.d_lpt[d] = static_cast<uint16_t>(r - out.tile_pbeg[t]);
    }
    // dummies repeat the tile's last camera so camera runs are unaffected
    for (uint32_t j = out.tile_ecnt[t]; j < out.tile_ebeg[t + 1] - out.tile_ebeg[t]; ++j)
      out.d_cam[out.tile_ebeg[t] + j] = out.tile_ecnt[t] ? out.d_cam[out.tile_ebeg[t] + out.tile_ecnt[t] - 1] : 0;
  }

  // distinct cameras per tile (edges are camera-sorted inside a tile) and the
  // per-edge local camera index used by the normal-tile kernels
  out.d_lcam.assign(slot, 0);
  out.tile_cam_off.assign(out.ntiles + 1, 0);
  for (uint32_t t = 0; t < out.ntiles; ++t) {
    const uint32_t eb = out.tile_ebeg[t];
    uint32_t nl = 0;
    for (uint32_t j = 0; j < out.tile_ecnt[t]; ++j) {
      if (j == 0 || out.d_cam[eb + j] != out.d_cam[eb + j - 1]) {
        out.tile_cams.push_back(out.d_cam[eb + j]);
        ++nl;
      }
      out.d_lcam[eb + j] = static_cast<uint16_t>(std::min<uint32_t>(nl - 1, 0xffffu));
    }
    for (uint32_t j = out.tile_ecnt[t]; j < out.tile_ebeg[t + 1] - eb; ++j) out.d_lcam[eb + j] = nl ? nl - 1 : 0;
    out.tile_cam_off[t + 1] = out.tile_cam_off[t] + nl;
  }
  classify_tiles(out);

  // per-point slot lists (tile-local, ascending)
  out.pt_slot_off.assign(in.np + 1, 0);
  for (uint64_t i = 0; i < in.np; ++i) out.pt_slot_off[i + 1] = out.pt_slot_off[i] + deg[out.pt_order[i]];
  out.pt_slots.resize(na);
  {
    std::vector<uint32_t> cur(out.pt_slot_off.begin(), out.pt_slot_off.end() - 1);
    for (uint32_t t = 0; t < out.ntiles; ++t)
      for (uint32_t j = 0; j < out.tile_ecnt[t]; ++j) {
        const uint32_t r = out.tile_pbeg[t] + out.d_lpt[out.tile_ebeg[t] + j];
        out.pt_slots[cur[r]++] = static_cast<uint16_t>(j & 0xffffu);
      }
  }

  build_partial_plan(out);
}

}  // namespace gb

namespace gb {

void shard_bounds(const uint32_t* tile_ebeg, const uint32_t* tile_pbeg, uint32_t ntiles, int world, int rank,
                  uint32_t* tile0, uint32_t* tile1, uint32_t* point0, uint32_t* point1) {
  const uint64_t total = tile_ebeg[ntiles];
  auto bound = [&](int r) -> uint32_t {
    if (r <= 0) return 0;
    if (r >= world) return ntiles;
    const uint64_t target = total * static_cast<uint64_t>(r) / static_cast<uint64_t>(world);
    // first tile whose slot begin reaches the target
    return static_cast<uint32_t>(std::lower_bound(tile_ebeg, tile_ebeg + ntiles, target) - tile_ebeg);
  };
  *tile0 = bound(rank);
  *tile1 = std::max(*tile0, bound(rank + 1));
  *point0 = tile_pbeg[*tile0];
  *point1 = tile_pbeg[*tile1];
}

void shard_range(const Activation& full, int world, int rank, uint32_t* tile0, uint32_t* tile1, uint32_t* point0,
                 uint32_t* point1) {
  shard_bounds(full.tile_ebeg.data(), full.tile_pbeg.data(), full.ntiles, world, rank, tile0, tile1, point0, point1);
}

void shard(const Activation& full, int world, int rank, Activation& out) {
  if (world <= 1) {
    out = full;
    return;
  }
  uint32_t t0, t1, p0, p1;
  shard_range(full, world, rank, &t0, &t1, &p0, &p1);
  out = Activation();
  out.nc = full.nc;
  out.np = p1 - p0;
  out.n_active = full.n_active;
  out.active = full.active;
  out.level = full.level;
  out.free_cams = full.free_cams;
  out.free_pts = full.free_pts;
  out.free_dims = full.free_dims;
  out.cam_col = full.cam_col;
  out.pt_col = full.pt_col;
  out.cam_inc = full.cam_inc;
  out.pt_inc = full.pt_inc;
  out.pt_order.assign(full.pt_order.begin() + p0, full.pt_order.begin() + p1);
  out.pt_rank = full.pt_rank;  // global internal ranks (debug surface only)
  out.ntiles = t1 - t0;
  const uint32_t s0 = full.tile_ebeg[t0], s1 = full.tile_ebeg[t1];
  out.n_slots = s1 - s0;
  for (uint32_t t = t0; t <= t1; ++t) {
    out.tile_ebeg.push_back(full.tile_ebeg[t] - s0);
    out.tile_pbeg.push_back(full.tile_pbeg[t] - p0);
    out.tile_cam_off.push_back(full.tile_cam_off[t] - full.tile_cam_off[t0]);
  }
  out.tile_ecnt.assign(full.tile_ecnt.begin() + t0, full.tile_ecnt.begin() + t1);
  out.tile_cams.assign(full.tile_cams.begin() + full.tile_cam_off[t0], full.tile_cams.begin() + full.tile_cam_off[t1]);
  for (uint32_t t : full.normal_tiles)
    if (t >= t0 && t < t1) out.normal_tiles.push_back(t - t0);
  for (uint32_t t : full.heavy_tiles)
    if (t >= t0 && t < t1) out.heavy_tiles.push_back(t - t0);
  out.d_a.assign(full.d_a.begin() + s0, full.d_a.begin() + s1);
  out.d_cam.assign(full.d_cam.begin() + s0, full.d_cam.begin() + s1);
  out.d_lpt.assign(full.d_lpt.begin() + s0, full.d_lpt.begin() + s1);
  out.d_lcam.assign(full.d_lcam.begin() + s0, full.d_lcam.begin() + s1);
  const uint32_t q0 = full.pt_slot_off[p0];
  for (uint32_t i = p0; i <= p1; ++i) out.pt_slot_off.push_back(full.pt_slot_off[i] - q0);
  out.pt_slots.assign(full.pt_slots.begin() + q0, full.pt_slots.begin() + full.pt_slot_off[p1]);
  build_partial_plan(out);
}

}  // namespace gb

namespace gb {
void build_incidence_host(uint64_t nvert, const std::vector<uint32_t>& vert_of_a, const uint8_t* fixed, Incidence& inc) {
  build_incidence(nvert, vert_of_a, fixed, inc);
}
}  // namespace gb
