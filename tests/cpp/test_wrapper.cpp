// C++ host-side test of include/cmgpu/cheesemap_gpu.hpp, written the way the
// reference's own tests are (tests/test_search.cpp:161-188 compares
// kernel_search against a linear scan; test_map.cpp:213-223 the dense cap).
// Built and run by tests/test_gpu_cpp.py on a GPU box.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <random>

#include "cmgpu/cheesemap_gpu.hpp"

namespace cg = cheesemap::gpu;

#define EXPECT(c)                                                   \
  do {                                                              \
    if (!(c)) {                                                     \
      std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #c); \
      std::exit(1);                                                 \
    }                                                               \
  } while (0)

static double sq(const cg::Point3& a, const cg::Point3& b) {
  const double dx = a.x - b.x, dy = a.y - b.y, dz = a.z - b.z;
  return dx * dx + dy * dy + dz * dz;
}

int main() {
  std::mt19937_64 eng(7);
  auto u = [&](double lo, double hi) {
    return lo + (hi - lo) * (static_cast<double>(eng() >> 11) * 0x1.0p-53);
  };
  cg::PointCloud cloud(20000);
  for (auto& p : cloud) p = {u(0, 40), u(0, 30), u(0, 10)};

  for (cg::Flavor f : {cg::Flavor::Dense, cg::Flavor::Sparse, cg::Flavor::Mixed}) {
    cg::BuildOptions o;
    o.flavor = f;
    const cg::Cheesemap map = cg::Cheesemap::build(cloud, o);
    EXPECT(map.size() == cloud.size());
    const cg::GridParams g = map.grid();
    EXPECT(g.nx == 40 || g.nx == 41);
    for (int t = 0; t < 40; ++t) {
      const cg::Point3 c{u(-2, 42), u(-2, 32), u(-2, 12)};
      const double r = u(0.1, 3.0);
      const auto got = cg::kernel_search(map, cg::SphereKernel{c, r});
      std::vector<cg::PointHandle> want;
      for (std::size_t h = 0; h < cloud.size(); ++h)
        if (sq(cloud[h], c) <= r * r) want.push_back(h);
      EXPECT(got == want);
      const auto knn = cg::knn_search(map, c, 10);
      std::vector<std::pair<double, std::size_t>> all;
      for (std::size_t h = 0; h < cloud.size(); ++h) all.push_back({sq(cloud[h], c), h});
      std::sort(all.begin(), all.end());
      EXPECT(knn.size() == 10);
      for (int i = 0; i < 10; ++i) EXPECT(knn[i].handle == all[i].second);
    }
  }
  // errors keep the reference's exception types
  bool threw = false;
  try {
    cg::Cheesemap::build({});
  } catch (const cg::EmptyCloudError&) {
    threw = true;
  }
  EXPECT(threw);
  threw = false;
  try {
    cg::BuildOptions o;
    o.dense_voxel_cap = 10;
    cg::Cheesemap::build(cloud, o);
  } catch (const cg::CapacityError&) {
    threw = true;
  }
  EXPECT(threw);
  std::printf("cpp wrapper ok\n");
  return 0;
}
