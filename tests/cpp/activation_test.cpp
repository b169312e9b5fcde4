// Host-side invariants of graph activation and sharding (activate.cpp),
// built with AddressSanitizer by tests/test_activation_cpu.py. Exit code 0 = ok.
#include <cstdio>
#include <cstdlib>
#include <random>
#include <set>
#include <vector>

#include "activate.hpp"

extern "C" int gb_synthetic_bal(uint64_t, uint64_t, uint64_t, uint64_t, uint64_t, double, uint32_t*, uint32_t*,
                                double*, double*, double*);

#define REQUIRE(c)                                                    \
  do {                                                                \
    if (!(c)) {                                                       \
      std::fprintf(stderr, "FAILED %s at line %d\n", #c, __LINE__); \
      std::exit(1);                                                   \
    }                                                                 \
  } while (0)

static void check(const gb::Activation& a, uint64_t np_local, bool sharded) {
  REQUIRE(a.tile_ebeg.size() == a.ntiles + 1u && a.tile_pbeg.size() == a.ntiles + 1u);
  REQUIRE(a.tile_ebeg.back() == a.n_slots && a.tile_pbeg.back() == np_local);
  REQUIRE(a.d_a.size() == a.n_slots && a.d_cam.size() == a.n_slots && a.d_lcam.size() == a.n_slots);
  REQUIRE(a.pt_order.size() == np_local && a.pt_slot_off.size() == np_local + 1);
  uint64_t real = 0;
  for (uint32_t t = 0; t < a.ntiles; ++t) {
    REQUIRE(a.tile_ebeg[t] % gb::kEdgePad == 0);
    REQUIRE(a.tile_ebeg[t] % gb::kJBlock == 0);  // one J store block per normal tile
    REQUIRE(a.tile_ebeg[t + 1] - a.tile_ebeg[t] == (a.tile_ecnt[t] + gb::kJBlock - 1) / gb::kJBlock * gb::kJBlock);
    REQUIRE(a.tile_ebeg[t] + a.tile_ecnt[t] <= a.tile_ebeg[t + 1]);
    real += a.tile_ecnt[t];
    const uint32_t npt = a.tile_pbeg[t + 1] - a.tile_pbeg[t];
    for (uint32_t j = 0; j < a.tile_ecnt[t]; ++j) {
      const uint32_t d = a.tile_ebeg[t] + j;
      REQUIRE(a.d_a[d] != gb::kNoKey && a.d_a[d] < a.active.size());
      REQUIRE(a.d_lpt[d] < npt || a.tile_ecnt[t] > gb::kTileEdges);
      REQUIRE(a.d_cam[d] < a.nc);
      REQUIRE(a.tile_cams[a.tile_cam_off[t] + a.d_lcam[d]] == a.d_cam[d]);
      if (j) REQUIRE(a.d_cam[d] >= a.d_cam[d - 1]);
    }
  }
  REQUIRE(real == a.pt_slots.size());
  REQUIRE(a.pt_slot_off.back() == a.pt_slots.size());
  REQUIRE(a.chunk_part_base.size() == a.nchunks + 1u && a.chunk_part_base.back() == a.nparts);
  REQUIRE(a.cam_part_off.size() == a.nc + 1 && a.cam_part_off.back() == a.nparts);
  std::vector<int> seen(a.nparts, 0);
  for (uint32_t q : a.cam_part_idx) {
    REQUIRE(q < a.nparts);
    seen[q]++;
  }
  for (int v : seen) REQUIRE(v == 1);
  (void)sharded;
}

int main() {
  const uint64_t shapes[][3] = {{49, 7776, 31843}, {520, 30, 15600}, {24, 600, 3600}, {8, 60, 300}};
  for (const auto& sh : shapes) {
    const uint64_t nc = sh[0], np = sh[1], ne = sh[2];
    std::vector<uint32_t> cam(ne), pt(ne);
    std::vector<double> obs(2 * ne), cams(9 * nc), pts(3 * np);
    REQUIRE(gb_synthetic_bal(nc, np, ne, 42, 0, 0.0, cam.data(), pt.data(), obs.data(), cams.data(), pts.data()) == 0);
    std::vector<uint8_t> level(ne, 0), cfix(nc, 0), pfix(np, 0);
    std::mt19937 rng(7);
    for (auto& l : level) l = (rng() % 20 == 0);
    for (auto& f : pfix) f = (rng() % 15 == 0);
    cfix[0] = 1;
    gb::ActivationInput in;
    in.nc = nc;
    in.np = np;
    in.ne = ne;
    in.cam = cam.data();
    in.pt = pt.data();
    in.level = level.data();
    in.cam_fixed = cfix.data();
    in.pt_fixed = pfix.data();
    gb::Activation full;
    gb::activate(in, full);
    check(full, np, false);
    for (int world : {2, 3, 5}) {
      uint64_t pts_total = 0, edges_total = 0;
      std::set<uint32_t> owned;
      for (int r = 0; r < world; ++r) {
        gb::Activation loc;
        gb::shard(full, world, r, loc);
        check(loc, loc.np, true);
        pts_total += loc.np;
        edges_total += loc.pt_slots.size();
        for (uint32_t p : loc.pt_order) REQUIRE(owned.insert(p).second);
      }
      REQUIRE(pts_total == np && owned.size() == np && edges_total == full.pt_slots.size());
    }
  }
  std::printf("activation invariants ok\n");
  return 0;
}
