#include <cstring>
#include <cstdio>
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
  // read_las: a hand-assembled LAS 1.2 file (test_io.cpp:58-72's values)
  {
    std::vector<unsigned char> b(227 + 2 * 20, 0);
    std::memcpy(b.data(), "LASF", 4);
    b[24] = 1, b[25] = 2;
    auto put16 = [&](size_t o, uint16_t v) { std::memcpy(&b[o], &v, 2); };
    auto put32 = [&](size_t o, uint32_t v) { std::memcpy(&b[o], &v, 4); };
    auto putd = [&](size_t o, double v) { std::memcpy(&b[o], &v, 8); };
    put16(94, 227), put32(96, 227), put16(105, 20), put32(107, 2);
    for (int a = 0; a < 3; ++a) putd(131 + 8 * a, 0.01), putd(155 + 8 * a, 100.0);
    const int32_t raw[6] = {12345, -200, 0, 0, 1, 2};
    for (int i = 0; i < 2; ++i) std::memcpy(&b[227 + 20 * i], raw + 3 * i, 12);
    const char* path = "/tmp/cmgpu_wrapper_test.las";
    FILE* f = std::fopen(path, "wb");
    std::fwrite(b.data(), 1, b.size(), f);
    std::fclose(f);
    const cg::LasFile lf = cg::read_las(path);
    EXPECT(lf.cloud.size() == 2 && lf.header.point_count == 2 && lf.header.scale_x == 0.01);
    EXPECT(lf.cloud[0].x == 12345 * 0.01 + 100.0 && lf.cloud[0].y == -200 * 0.01 + 100.0);
    EXPECT(lf.cloud[1].z == 2 * 0.01 + 100.0);
    threw = false;
    try {
      cg::read_las("/tmp/cmgpu_wrapper_missing.las");
    } catch (const cg::IoError&) {
      threw = true;
    }
    EXPECT(threw);
    b[0] = 'X';
    f = std::fopen(path, "wb");
    std::fwrite(b.data(), 1, b.size(), f);
    std::fclose(f);
    threw = false;
    try {
      cg::read_las(path);
    } catch (const cg::ParseError&) {
      threw = true;
    }
    EXPECT(threw);
    std::remove(path);
  }
  std::printf("cpp wrapper ok\n");
  return 0;
}
