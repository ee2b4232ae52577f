// TEST INFRASTRUCTURE — C-ABI adapter over the UNMODIFIED reference library.
//
// Compiled (oracle/Makefile) together with the reference's own sources,
// read in place from /root/reference/proj/core, into oracle/_ref/libcheesemap_ref.so.
// Nothing here re-implements the algorithm: every call goes through the
// reference's public API (Cheesemap::build, kernel_search, knn_search,
// occupancy_stats, voxel_lookup). Used to pin the CPU restatement
// (oracle/cheesemap_oracle.cpp), to generate tests/golden/, and as the CPU
// baseline / `bench.py --impl reference` arm.
//
// The exported functions mirror oracle/cheesemap_oracle.cpp's orc_* ABI so
// the two are interchangeable in tests.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "cheesemap/analysis.hpp"
#include "cheesemap/io.hpp"
#include "cheesemap/map.hpp"
#include "cheesemap/search.hpp"

using namespace cheesemap;

struct ref_index {
  PointCloud cloud;  // the map borrows the cloud (map.hpp:50-52)
  std::optional<Cheesemap> map;
};

namespace {

int status_of(const std::exception& e) {
  if (dynamic_cast<const EmptyCloudError*>(&e)) return 1;
  if (dynamic_cast<const InvalidArgumentError*>(&e)) return 2;
  if (dynamic_cast<const CapacityError*>(&e)) return 3;
  if (dynamic_cast<const OutOfDomainError*>(&e)) return 4;
  if (dynamic_cast<const ParseError*>(&e)) return 7;
  if (dynamic_cast<const IoError*>(&e)) return 8;
  return 99;
}

template <class F>
void parallel_queries(std::uint64_t nq, unsigned threads, F&& f) {
  if (threads == 0) threads = std::max(1u, std::thread::hardware_concurrency());
  threads = static_cast<unsigned>(std::min<std::uint64_t>(threads, std::max<std::uint64_t>(nq, 1)));
  if (threads <= 1) {
    for (std::uint64_t q = 0; q < nq; ++q) f(q);
    return;
  }
  std::vector<std::thread> pool;
  for (unsigned t = 0; t < threads; ++t)
    pool.emplace_back([&, t] {
      for (std::uint64_t q = t; q < nq; q += threads) f(q);
    });
  for (auto& th : pool) th.join();
}

std::uint64_t mix64(std::uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

// The kNN restatement's bound kernel: the reference's Kernel
// concept (geometry.hpp:67-71) with is_inside = d^2 <= D.
struct D2Kernel {
  Point3 c;
  double d2max;
  double half;
  Aabb box() const {
    return {{c.x - half, c.y - half, c.z - half}, {c.x + half, c.y + half, c.z + half}};
  }
  bool is_inside(const Point3& p) const { return squared_distance(p, c) <= d2max; }
};
static_assert(Kernel<D2Kernel>);

struct NoneKernel {
  Aabb b;
  Aabb box() const { return b; }
  bool is_inside(const Point3&) const { return false; }
};

std::vector<PointHandle> run_kernel(const Cheesemap& m, int kernel, const Point3& c, double r,
                                    QueryStats* st) {
  if (kernel == 0) return kernel_search(m, SphereKernel{c, r}, st);
  if (kernel == 2) {
    CylinderKernel k;
    k.center_x = c.x;
    k.center_y = c.y;
    k.radius = r;
    return kernel_search(m, k, st);
  }
  const Aabb b{{c.x - r, c.y - r, c.z - r}, {c.x + r, c.y + r, c.z + r}};
  return kernel_search(m, BoxKernel{b}, st);
}

}  // namespace

extern "C" {

// The reference's own UniformBox generator (io.cpp:252-272), to pin the RNG
// conventions the BASELINE-config generators reuse.
int ref_generate_uniform(uint64_t seed, uint64_t n, double ex, double ey, double ez, double* out) {
  SyntheticSpec spec;
  spec.kind = SyntheticSpec::Kind::UniformBox;
  spec.count = n;
  spec.extent_x = ex;
  spec.extent_y = ey;
  spec.extent_z = ez;
  spec.seed = seed;
  try {
    const PointCloud c = generate(spec);
    std::memcpy(out, c.data(), n * sizeof(Point3));
  } catch (const std::exception& e) {
    return status_of(e);
  }
  return 0;
}

int ref_build(const double* xyz, uint64_t n, int flavor, int mode, double cx, double cy,
              double cz, double tau, uint64_t dense_cap, ref_index** out) {
  *out = nullptr;
  auto r = new ref_index();
  r->cloud.resize(n);
  if (n) std::memcpy(r->cloud.data(), xyz, n * sizeof(Point3));
  BuildOptions o;
  o.flavor = static_cast<Flavor>(flavor);
  o.mode = mode ? GridMode::ThreeD : GridMode::TwoD;
  o.cell = {cx, cy, cz};
  o.reorder = false;
  o.densify_threshold = tau;
  o.dense_voxel_cap = dense_cap;
  try {
    r->map.emplace(Cheesemap::build(r->cloud, o));
  } catch (const std::exception& e) {
    delete r;
    return status_of(e);
  }
  *out = r;
  return 0;
}

void ref_free(ref_index* r) { delete r; }

void ref_grid(const ref_index* r, double* origin3, double* cell3, uint64_t* dims3,
              double* bmin3, double* bmax3) {
  const GridParams& g = r->map->grid();
  origin3[0] = g.origin.x, origin3[1] = g.origin.y, origin3[2] = g.origin.z;
  cell3[0] = g.cell.x, cell3[1] = g.cell.y, cell3[2] = g.cell.z;
  dims3[0] = g.nx, dims3[1] = g.ny, dims3[2] = g.nz;
  bmin3[0] = g.bounds.min.x, bmin3[1] = g.bounds.min.y, bmin3[2] = g.bounds.min.z;
  bmax3[0] = g.bounds.max.x, bmax3[1] = g.bounds.max.y, bmax3[2] = g.bounds.max.z;
}

uint64_t ref_non_empty(const ref_index* r) { return r->map->occupancy_stats().non_empty; }

void ref_memory_report(const ref_index* r, uint64_t* out3) {
  const MemoryReport m = r->map->memory_report();
  out3[0] = m.handle_bytes;
  out3[1] = m.structure_bytes;
  out3[2] = m.total_bytes;
}

uint64_t ref_slice_flags(const ref_index* r, uint8_t* dense, uint64_t* non_empty) {
  const OccupancyStats st = r->map->occupancy_stats();
  for (std::size_t k = 0; k < st.slices.size(); ++k) {
    if (dense) dense[k] = st.slices[k].dense;
    if (non_empty) non_empty[k] = st.slices[k].non_empty;
  }
  return st.slices.size();
}

// (key, handle) grouped by voxel in ascending key order, handles in the
// order voxel_lookup returns them (map.cpp:138-148).
void ref_export(const ref_index* r, uint64_t* keys, uint64_t* handles) {
  const GridParams& g = r->map->grid();
  std::vector<std::uint64_t> vk(r->cloud.size());
  for (std::size_t h = 0; h < r->cloud.size(); ++h) vk[h] = g.global_index(g.voxel_of(r->cloud[h]));
  std::sort(vk.begin(), vk.end());
  vk.erase(std::unique(vk.begin(), vk.end()), vk.end());
  std::uint64_t pos = 0;
  for (std::uint64_t key : vk) {
    const auto list = r->map->voxel_lookup(g.coord_of(key));
    for (PointHandle h : *list) {
      if (keys) keys[pos] = key;
      if (handles) handles[pos] = h;
      ++pos;
    }
  }
}

int ref_radius(const ref_index* r, const double* q, uint64_t nq, int kernel, double rad,
               unsigned threads, uint32_t* counts, uint64_t* digests, uint64_t* points_tested,
               uint64_t* voxels_visited) {
  if (kernel < 0 || kernel > 2) return 2;
  parallel_queries(nq, threads, [&](std::uint64_t qi) {
    QueryStats st;
    const auto res = run_kernel(*r->map, kernel, {q[3 * qi], q[3 * qi + 1], q[3 * qi + 2]}, rad, &st);
    if (counts) counts[qi] = static_cast<uint32_t>(res.size());
    if (digests) {
      std::uint64_t d = 0;
      for (PointHandle h : res) d += mix64(h);
      digests[qi] = d;
    }
    if (points_tested) points_tested[qi] = st.points_tested;
    if (voxels_visited) voxels_visited[qi] = st.voxels_visited;
  });
  return 0;
}

int ref_radius_fill(const ref_index* r, const double* q, uint64_t nq, int kernel, double rad,
                    unsigned threads, const uint64_t* row_ptr, uint32_t* cols) {
  if (kernel < 0 || kernel > 2) return 2;
  parallel_queries(nq, threads, [&](std::uint64_t qi) {
    auto res = run_kernel(*r->map, kernel, {q[3 * qi], q[3 * qi + 1], q[3 * qi + 2]}, rad, nullptr);
    std::sort(res.begin(), res.end());  // tests/test_util.hpp:30-35
    for (std::size_t t = 0; t < res.size(); ++t) cols[row_ptr[qi] + t] = static_cast<uint32_t>(res[t]);
  });
  return 0;
}

// kNN restatement over the reference's knn_search.
int ref_knn(const ref_index* r, const double* q, uint64_t nq, uint32_t k, unsigned threads,
            uint32_t* idx_out, double* d2_out, uint64_t* points_tested_rk,
            uint64_t* points_tested_alg2) {
  if (k == 0) return 2;
  parallel_queries(nq, threads, [&](std::uint64_t qi) {
    const Point3 c{q[3 * qi], q[3 * qi + 1], q[3 * qi + 2]};
    QueryStats st;
    const auto found = knn_search(*r->map, c, k, GrowthPolicy::Density, &st);
    if (points_tested_alg2) points_tested_alg2[qi] = st.points_tested;
    double D = 0.0;
    for (const Neighbor& nb : found) D = std::max(D, squared_distance(r->cloud[nb.handle], c));
    const D2Kernel kern{c, D, std::sqrt(D) * (1.0 + 1e-9) + 1e-300};
    const auto all = kernel_search(*r->map, kern);
    std::vector<std::pair<double, PointHandle>> v;
    v.reserve(all.size());
    for (PointHandle h : all) v.push_back({squared_distance(r->cloud[h], c), h});
    std::sort(v.begin(), v.end());
    for (uint32_t t = 0; t < k; ++t) {
      idx_out[qi * k + t] = t < v.size() ? static_cast<uint32_t>(v[t].second) : UINT32_MAX;
      if (d2_out) d2_out[qi * k + t] = t < v.size() ? v[t].first : INFINITY;
    }
    if (points_tested_rk) {
      const double dk = v.empty() ? 0.0 : std::sqrt(v[std::min<std::size_t>(k, v.size()) - 1].first);
      QueryStats s3;
      kernel_search(*r->map, NoneKernel{{{c.x - dk, c.y - dk, c.z - dk}, {c.x + dk, c.y + dk, c.z + dk}}}, &s3);
      points_tested_rk[qi] = s3.points_tested;
    }
  });
  return 0;
}

// The reference's own weighted_density (analysis.cpp:26-86).
int ref_weighted_density(const double* xyz, uint64_t n, uint64_t sample_size, uint64_t seed,
                         unsigned /*threads*/, double* value, uint64_t* bins256) {
  PointCloud cloud(n);
  if (n) std::memcpy(cloud.data(), xyz, n * sizeof(Point3));
  try {
    const WeightedDensity wd = sample_size ? weighted_density(cloud, sample_size, seed)
                                           : weighted_density(cloud);
    *value = wd.value;
    for (int b = 0; b < 256; ++b) bins256[b] = wd.histogram.bins[b];
  } catch (const std::exception& e) {
    return status_of(e);
  }
  return 0;
}

// read_las / write_las through the reference (io.cpp:33-166). The header
// struct has orc_las_header's layout. Status as status_of; `msg` gets what().
struct ref_las_header {
  uint8_t version_major, version_minor, point_format;
  uint16_t header_size, record_length;
  uint32_t data_offset;
  uint64_t point_count;
  double scale[3], offset[3];
  double bounds_min[3], bounds_max[3];
};

static void copy_msg(char* msg, int msglen, const char* m) {
  if (msg && msglen > 0) {
    std::strncpy(msg, m, (size_t)msglen - 1);
    msg[msglen - 1] = 0;
  }
}

int ref_las_read(const char* path, ref_las_header* h, double* xyz, uint64_t cap, char* msg,
                 int msglen) {
  try {
    const LasFile f = read_las(path);
    std::memset(h, 0, sizeof(*h));
    h->version_major = f.header.version_major;
    h->version_minor = f.header.version_minor;
    h->point_format = f.header.point_format;
    h->point_count = f.header.point_count;
    h->scale[0] = f.header.scale_x, h->scale[1] = f.header.scale_y, h->scale[2] = f.header.scale_z;
    h->offset[0] = f.header.offset_x, h->offset[1] = f.header.offset_y,
    h->offset[2] = f.header.offset_z;
    h->bounds_min[0] = f.header.bounds.min.x, h->bounds_min[1] = f.header.bounds.min.y,
    h->bounds_min[2] = f.header.bounds.min.z;
    h->bounds_max[0] = f.header.bounds.max.x, h->bounds_max[1] = f.header.bounds.max.y,
    h->bounds_max[2] = f.header.bounds.max.z;
    if (xyz) {
      if (f.cloud.size() > cap) return 2;
      std::memcpy(xyz, f.cloud.data(), f.cloud.size() * sizeof(Point3));
    }
  } catch (const std::exception& e) {
    copy_msg(msg, msglen, e.what());
    return status_of(e);
  }
  return 0;
}

int ref_las_write(const double* xyz, uint64_t n, const char* path, double scale, char* msg,
                  int msglen) {
  try {
    PointCloud c(n);
    if (n) std::memcpy(c.data(), xyz, n * sizeof(Point3));
    write_las(c, path, scale);
  } catch (const std::exception& e) {
    copy_msg(msg, msglen, e.what());
    return status_of(e);
  }
  return 0;
}

// parse_synthetic_spec + generate through the reference (io.cpp:252-399):
// returns the count in *n_out; xyz (capacity cap points) may be null.
int ref_generate_spec(const char* text, double* xyz, uint64_t cap, uint64_t* n_out, char* msg,
                      int msglen) {
  try {
    const PointCloud c = generate(parse_synthetic_spec(text));
    *n_out = c.size();
    if (xyz) {
      if (c.size() > cap) return 2;
      std::memcpy(xyz, c.data(), c.size() * sizeof(Point3));
    }
  } catch (const std::exception& e) {
    copy_msg(msg, msglen, e.what());
    return status_of(e);
  }
  return 0;
}

}  // extern "C"
