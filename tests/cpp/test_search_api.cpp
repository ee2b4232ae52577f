// The reference's search API as its own tests use it (tests/test_search.cpp
// "kernel search against the linear-scan oracle" and "kernel search edge
// cases", test_map.cpp voxel_lookup / memory_report), against
// cheesemap::gpu: general BoxKernel{Aabb} boxes, bounded and unbounded
// CylinderKernels, QueryStats, GrowthPolicy, voxel_present / voxel_lookup,
// memory_report, and the reference exception types. Built and run by
// tests/test_gpu_cpp.py on a GPU box.
#include <cstdio>
#include <cstdlib>
#include <random>

#include "cmgpu/cheesemap_gpu.hpp"

using namespace cheesemap::gpu;

#define EXPECT(c)                                                          \
  do {                                                                     \
    if (!(c)) {                                                            \
      std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #c); \
      std::exit(1);                                                        \
    }                                                                      \
  } while (0)

static PointCloud box_cloud(std::size_t n, double ex, double ey, double ez, std::uint64_t seed) {
  std::mt19937_64 eng(seed);
  auto u = [&](double lo, double hi) {
    return lo + (hi - lo) * (static_cast<double>(eng() >> 11) * 0x1.0p-53);
  };
  PointCloud c(n);
  for (auto& p : c) p = {u(0, ex), u(0, ey), u(0, ez)};
  return c;
}

static Cheesemap make(const PointCloud& cloud, Flavor f, GridMode m, double cell) {
  BuildOptions o;
  o.flavor = f;
  o.mode = m;
  o.cell = CellSize::uniform(cell);
  return Cheesemap::build(cloud, o);
}

int main() {
  const PointCloud cloud = box_cloud(4000, 25, 25, 12, 21);
  std::vector<Cheesemap> maps;
  for (const Flavor f : {Flavor::Dense, Flavor::Sparse, Flavor::Mixed})
    for (const GridMode m : {GridMode::TwoD, GridMode::ThreeD})
      for (const double cell : {0.5, 1.0, 2.5}) maps.push_back(make(cloud, f, m, cell));
  std::mt19937_64 eng(43);
  for (int q = 0; q < 25; ++q) {
    const Point3 c = cloud[eng() % cloud.size()];
    const double r = 0.3 + 5.7 * (static_cast<double>(eng() >> 11) * 0x1.0p-53);
    const SphereKernel sphere{c, r};
    const BoxKernel cube{{{c.x - r, c.y - r, c.z - r}, {c.x + r, c.y + r, c.z + r}}};
    // a non-cubic box and a bounded cylinder (the general forms)
    const BoxKernel slab{{{c.x - 2 * r, c.y - 0.5 * r, c.z - 0.25 * r}, {c.x + r, c.y + r, c.z + 3 * r}}};
    const CylinderKernel cyl{c.x, c.y, r};
    const CylinderKernel bounded{c.x, c.y, r, c.z - 1.0, c.z + 0.5};
    const auto ws = brute_radius(cloud, sphere), wc = brute_radius(cloud, cube),
               wb = brute_radius(cloud, slab), wy = brute_radius(cloud, cyl),
               wz = brute_radius(cloud, bounded);
    for (const Cheesemap& map : maps) {
      EXPECT(kernel_search(map, sphere) == ws);
      EXPECT(kernel_search(map, cube) == wc);
      EXPECT(kernel_search(map, slab) == wb);
      EXPECT(kernel_search(map, cyl) == wy);
      EXPECT(kernel_search(map, bounded) == wz);
    }
  }
  // edge cases with stats (test_search.cpp "kernel search edge cases")
  {
    const PointCloud c2 = box_cloud(1000, 10, 10, 10, 2);
    const Cheesemap map = make(c2, Flavor::Dense, GridMode::ThreeD, 1.0);
    QueryStats st;
    const auto none = kernel_search(map, SphereKernel{{100, 100, 100}, 1.0}, &st);
    EXPECT(none.empty() && st.voxels_visited == 0 && st.points_tested == 0);
    const auto all = kernel_search(map, SphereKernel{{5, 5, 5}, 100.0}, &st);
    EXPECT(all.size() == c2.size());
    EXPECT(st.voxels_visited == map.grid().total_voxels());
    EXPECT(st.points_tested == c2.size());
    // knn with a policy and stats: exact, stats of the k-th-distance sphere
    const auto nn = knn_search(map, Point3{5, 5, 5}, 12, GrowthPolicy::Monotonic, &st);
    EXPECT(nn.size() == 12);
    for (std::size_t i = 1; i < nn.size(); ++i) EXPECT(nn[i - 1].distance <= nn[i].distance);
    EXPECT(st.final_radius == nn.back().distance && st.points_tested >= 12);
    // voxel_present / voxel_lookup / memory_report
    std::uint64_t seen = 0;
    const GridParams g = map.grid();
    for (std::uint64_t i = 0; i < g.nx; ++i)
      for (std::uint64_t j = 0; j < g.ny; ++j)
        for (std::uint64_t k = 0; k < g.nz; ++k) {
          EXPECT(map.voxel_present({i, j, k}));  // dense: always materialized
          const auto h = map.voxel_lookup({i, j, k});
          EXPECT(h.has_value());
          EXPECT(std::is_sorted(h->begin(), h->end()));
          seen += h->size();
        }
    EXPECT(seen == c2.size());
    const MemoryReport mr = map.memory_report();
    EXPECT(mr.handle_bytes == 8 * c2.size() && mr.total_bytes == mr.handle_bytes + mr.structure_bytes);
    const Cheesemap sp = make(c2, Flavor::Sparse, GridMode::ThreeD, 0.25);
    std::uint64_t absent = 0;
    for (std::uint64_t i = 0; i < 6; ++i) {
      const bool p = sp.voxel_present({i, 0, 0});
      const auto h = sp.voxel_lookup({i, 0, 0});
      EXPECT(p == h.has_value());
      absent += !p;
    }
    EXPECT(absent > 0);
    bool threw = false;
    try {
      (void)sp.voxel_lookup({1u << 30, 0, 0});
    } catch (const cheesemap::OutOfDomainError&) {
      threw = true;
    }
    EXPECT(threw);
  }
  // the reference's exception types, caught through namespace cheesemap
  bool threw = false;
  try {
    BuildOptions o;
    o.dense_voxel_cap = 10;
    Cheesemap::build(cloud, o);
  } catch (const cheesemap::CapacityError&) {
    threw = true;
  }
  EXPECT(threw);
  threw = false;
  try {
    Cheesemap::build({});
  } catch (const cheesemap::Error&) {
    threw = true;
  }
  EXPECT(threw);
  std::printf("cpp search api ok\n");
  return 0;
}
