// cheesemap_gpu.hpp — header-only C++ mirror of the reference's index API
// (/root/reference/proj/core/include/cheesemap/{geometry,grid,map,search,
// errors}.hpp) over the C ABI in cmgpu.h. A reference user switches by
// replacing `cheesemap::` with `cheesemap::gpu::` — same names, argument
// meaning and exception types — and gains the batched calls the reference
// lacks (radius_search, knn_batch, radius_digest).
//
// Differences a caller can observe:
//  * kernel_search returns handles sorted ascending (the reference returns
//    voxel-visit order, search.hpp:110-122; its tests sort,
//    tests/test_util.hpp:30-35);
//  * knn_search orders ties by handle (the reference keeps insertion order,
//    search.cpp:16-28); distances are sqrt of the same fp64 d^2. It is exact
//    for any GrowthPolicy (the policy only steers the reference's Alg. 2);
//    its QueryStats report the candidates of kernel_search at the exact k-th
//    distance (points_tested, voxels_visited), growth_iterations = 0 and
//    final_radius = that distance;
//  * the map owns device copies of the points (the cloud need not outlive it).
//
// Exceptions ARE the reference's: when <cheesemap/errors.hpp> is on the
// include path it is used directly; otherwise the same hierarchy is declared
// in namespace cheesemap (errors.hpp:8-42). Either way a caller's
// `catch (cheesemap::CapacityError&)` catches what this mirror throws.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../cmgpu.h"

#if __has_include(<cheesemap/errors.hpp>)
#include <cheesemap/errors.hpp>
#else
namespace cheesemap {
class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class EmptyCloudError : public Error {
 public:
  EmptyCloudError() : Error("point cloud is empty") {}
  using Error::Error;
};
class CapacityError : public Error { public: using Error::Error; };
class OutOfDomainError : public Error { public: using Error::Error; };
class ParseError : public Error { public: using Error::Error; };
class InvalidArgumentError : public Error { public: using Error::Error; };
class IoError : public Error { public: using Error::Error; };
}  // namespace cheesemap
#endif

namespace cheesemap::gpu {

// ------------------------------------------------------------ errors.hpp --
using ::cheesemap::CapacityError;
using ::cheesemap::EmptyCloudError;
using ::cheesemap::Error;
using ::cheesemap::InvalidArgumentError;
using ::cheesemap::IoError;
using ::cheesemap::OutOfDomainError;
using ::cheesemap::ParseError;
// device / collective failures (no reference analogue), still a cheesemap::Error
class CudaError : public ::cheesemap::Error { public: using ::cheesemap::Error::Error; };

inline void check(cm_status s) {
  if (s == CM_OK) return;
  const std::string msg = std::string(cm_status_name(s)) + ": " + cm_last_error();
  switch (s) {
    case CM_EMPTY_CLOUD: throw EmptyCloudError(msg);
    case CM_INVALID_ARGUMENT: throw InvalidArgumentError(msg);
    case CM_CAPACITY: throw CapacityError(msg);
    case CM_OUT_OF_DOMAIN: throw OutOfDomainError(msg);
    case CM_PARSE: throw ParseError(msg);
    case CM_IO: throw IoError(msg);
    default: throw CudaError(msg);
  }
}

// ---------------------------------------------------------- geometry.hpp --
struct Point3 {
  double x = 0.0, y = 0.0, z = 0.0;
};
static_assert(sizeof(Point3) == 24, "PointCloud layout is n x 3 doubles");
using PointHandle = std::uint64_t;
using PointCloud = std::vector<Point3>;

// Axis-aligned box, closed on all faces (geometry.hpp:43-58).
struct Aabb {
  Point3 min, max;
  bool contains(const Point3& p) const {
    return p.x >= min.x && p.x <= max.x && p.y >= min.y && p.y <= max.y && p.z >= min.z &&
           p.z <= max.z;
  }
  bool intersects(const Aabb& o) const {
    return min.x <= o.max.x && max.x >= o.min.x && min.y <= o.max.y && max.y >= o.min.y &&
           min.z <= o.max.z && max.z >= o.min.z;
  }
};

inline double squared_distance(const Point3& a, const Point3& b) {  // geometry.hpp:26-31
  const double dx = a.x - b.x, dy = a.y - b.y, dz = a.z - b.z;
  return dx * dx + dy * dy + dz * dz;
}

// The three kernels of geometry.hpp:73-113, with the reference's box() and
// is_inside() (the device applies the same arithmetic).
struct SphereKernel {
  Point3 center;
  double radius = 0.0;
  Aabb box() const {
    return {{center.x - radius, center.y - radius, center.z - radius},
            {center.x + radius, center.y + radius, center.z + radius}};
  }
  bool is_inside(const Point3& p) const { return squared_distance(p, center) <= radius * radius; }
};
struct BoxKernel {
  Aabb aabb;
  Aabb box() const { return aabb; }
  bool is_inside(const Point3& p) const { return aabb.contains(p); }
  // the cube the reference CLI builds (cmd_bench.cpp:107-111)
  static BoxKernel cube(const Point3& c, double r) {
    return {{{c.x - r, c.y - r, c.z - r}, {c.x + r, c.y + r, c.z + r}}};
  }
};
struct CylinderKernel {  // vertical, optional z range (geometry.hpp:97-113)
  double center_x = 0.0, center_y = 0.0, radius = 0.0;
  double z_lo = -std::numeric_limits<double>::infinity();
  double z_hi = std::numeric_limits<double>::infinity();
  Aabb box() const {
    return {{center_x - radius, center_y - radius, z_lo}, {center_x + radius, center_y + radius, z_hi}};
  }
  bool is_inside(const Point3& p) const {
    const double dx = p.x - center_x, dy = p.y - center_y;
    return p.z >= z_lo && p.z <= z_hi && dx * dx + dy * dy <= radius * radius;
  }
};

// ------------------------------------------------------ grid.hpp, map.hpp --
enum class GridMode { TwoD = CM_TWOD, ThreeD = CM_THREED };
enum class Flavor { Dense = CM_DENSE, Sparse = CM_SPARSE, Mixed = CM_MIXED };

struct CellSize {
  double x = 1.0, y = 1.0, z = 1.0;
  static CellSize uniform(double s) { return {s, s, s}; }
};

struct BuildOptions {
  Flavor flavor = Flavor::Dense;
  GridMode mode = GridMode::ThreeD;
  CellSize cell = CellSize::uniform(1.0);
  bool reorder = false;
  double densify_threshold = 0.80;
  std::uint64_t dense_voxel_cap = std::uint64_t{1} << 32;
};

struct GridParams {
  Point3 origin;
  CellSize cell;
  std::uint64_t nx = 1, ny = 1, nz = 1;
  GridMode mode = GridMode::ThreeD;
  Point3 bounds_min, bounds_max;
  std::uint64_t total_voxels() const { return nx * ny * nz; }
};

struct VoxelCoord {  // grid.hpp:21-27
  std::uint64_t i = 0, j = 0, k = 0;
};

struct MemoryReport {  // map.hpp:41-48
  std::uint64_t handle_bytes = 0;
  std::uint64_t structure_bytes = 0;
  std::uint64_t total_bytes = 0;
};

struct SliceOccupancy {
  bool dense = false;
  std::uint64_t cells = 0;
  std::uint64_t non_empty = 0;
};

struct OccupancyStats {
  std::uint64_t total_voxels = 0;
  std::uint64_t non_empty = 0;
  double empty_fraction = 0.0;
  std::vector<SliceOccupancy> slices;  // mixed flavour only, as the reference
};

struct QueryStats {  // search.hpp:12-17
  std::uint64_t voxels_visited = 0;
  std::uint64_t points_tested = 0;
  std::uint64_t growth_iterations = 0;
  double final_radius = 0.0;
};

enum class GrowthPolicy { Density, Monotonic };  // search.hpp:88

struct Neighbor {
  PointHandle handle = 0;
  double distance = 0.0;
};

// Sorted CSR neighbour lists of a batch of centres.
struct Csr {
  std::vector<std::uint64_t> row_ptr;  // nq + 1
  std::vector<std::uint32_t> cols;     // handles, ascending per row
};

class Cheesemap {
 public:
  static Cheesemap build(const PointCloud& cloud, const BuildOptions& opts = {},
                         int device = 0) {
    cm_build_options o;
    cm_default_options(&o);
    o.flavor = static_cast<int32_t>(opts.flavor);
    o.mode = static_cast<int32_t>(opts.mode);
    o.cell_x = opts.cell.x;
    o.cell_y = opts.cell.y;
    o.cell_z = opts.cell.z;
    o.reorder = opts.reorder ? 1 : 0;
    o.densify_threshold = opts.densify_threshold;
    o.dense_voxel_cap = opts.dense_voxel_cap;
    cm_index* h = nullptr;
    check(cm_build(reinterpret_cast<const double*>(cloud.data()), cloud.size(), &o, device,
                   nullptr, &h));
    return Cheesemap(h, opts);
  }

  Cheesemap(Cheesemap&& o) noexcept : h_(std::exchange(o.h_, nullptr)), opts_(o.opts_) {}
  Cheesemap& operator=(Cheesemap&& o) noexcept {
    if (this != &o) {
      cm_free(h_);
      h_ = std::exchange(o.h_, nullptr);
      opts_ = o.opts_;
    }
    return *this;
  }
  Cheesemap(const Cheesemap&) = delete;
  Cheesemap& operator=(const Cheesemap&) = delete;
  ~Cheesemap() { cm_free(h_); }

  GridParams grid() const {
    cm_grid_params g;
    check(cm_get_grid(h_, &g));
    GridParams p;
    p.origin = {g.origin[0], g.origin[1], g.origin[2]};
    p.cell = {g.cell[0], g.cell[1], g.cell[2]};
    p.nx = g.nx, p.ny = g.ny, p.nz = g.nz;
    p.mode = static_cast<GridMode>(g.mode);
    p.bounds_min = {g.bounds_min[0], g.bounds_min[1], g.bounds_min[2]};
    p.bounds_max = {g.bounds_max[0], g.bounds_max[1], g.bounds_max[2]};
    return p;
  }
  Flavor flavor() const { return opts_.flavor; }
  GridMode mode() const { return opts_.mode; }
  bool reordered() const { return opts_.reorder; }
  std::uint64_t size() const { return cm_size(h_); }

  OccupancyStats occupancy_stats() const {
    const std::uint64_t nz = grid().nz;
    std::vector<std::uint8_t> dense(nz);
    std::vector<std::uint64_t> ne(nz);
    cm_occupancy o;
    check(cm_get_occupancy(h_, &o, dense.data(), ne.data(), nz));
    OccupancyStats st;
    st.total_voxels = o.total_voxels;
    st.non_empty = o.non_empty;
    st.empty_fraction = o.empty_fraction;
    if (opts_.flavor == Flavor::Mixed) {
      const GridParams g = grid();
      for (std::uint64_t k = 0; k < nz; ++k) st.slices.push_back({dense[k] != 0, g.nx * g.ny, ne[k]});
    }
    return st;
  }

  // map.hpp:62-69: materialized? (dense: always; mixed: any cell of a
  // densified slice; else non-empty) and the voxel's handles (ascending)
  bool voxel_present(const VoxelCoord& v) const {
    int present = 0;
    std::uint64_t n = 0;
    check(cm_voxel_lookup(h_, v.i, v.j, v.k, &present, nullptr, 0, &n));
    return present != 0;
  }
  std::optional<std::vector<PointHandle>> voxel_lookup(const VoxelCoord& v) const {
    int present = 0;
    std::uint64_t n = 0;
    check(cm_voxel_lookup(h_, v.i, v.j, v.k, &present, nullptr, 0, &n));
    if (!present) return std::nullopt;
    std::vector<std::uint32_t> h(n);
    if (n) check(cm_voxel_lookup(h_, v.i, v.j, v.k, &present, h.data(), n, &n));
    return std::vector<PointHandle>(h.begin(), h.end());
  }
  MemoryReport memory_report() const {  // map.hpp:105, map.cpp:173-192
    cm_memory_report r;
    check(cm_get_memory_report(h_, &r));
    return {r.handle_bytes, r.structure_bytes, r.total_bytes};
  }
  std::uint64_t device_bytes() const {
    cm_memory_report r;
    check(cm_get_memory_report(h_, &r));
    return r.device_bytes;
  }

  void corrupt_for_testing() { check(cm_corrupt_for_testing(h_)); }
  const cm_index* handle() const { return h_; }

 private:
  Cheesemap(cm_index* h, const BuildOptions& o) : h_(h), opts_(o) {}
  cm_index* h_ = nullptr;
  BuildOptions opts_;
};

// ------------------------------------------------------------ search.hpp --
inline Csr radius_search(const Cheesemap& m, const std::vector<Point3>& centers, double r,
                         cm_kernel kind = CM_SPHERE) {
  cm_csr* csr = nullptr;
  check(cm_radius_search(m.handle(), reinterpret_cast<const double*>(centers.data()),
                         centers.size(), kind, r, nullptr, &csr));
  std::uint64_t nq = 0, nnz = 0;
  cm_csr_info(csr, &nq, &nnz, nullptr, nullptr);
  Csr out;
  out.row_ptr.resize(nq + 1);
  out.cols.resize(nnz);
  const cm_status s = cm_csr_download(csr, out.row_ptr.data(), out.cols.data(), nullptr);
  cm_csr_free(csr);
  check(s);
  return out;
}

namespace detail {
inline void kernel_params(const SphereKernel& k, std::vector<double>& p) {
  p.insert(p.end(), {k.center.x, k.center.y, k.center.z, k.radius});
}
inline void kernel_params(const BoxKernel& k, std::vector<double>& p) {
  p.insert(p.end(), {k.aabb.min.x, k.aabb.min.y, k.aabb.min.z, k.aabb.max.x, k.aabb.max.y,
                     k.aabb.max.z});
}
inline void kernel_params(const CylinderKernel& k, std::vector<double>& p) {
  p.insert(p.end(), {k.center_x, k.center_y, k.radius, k.z_lo, k.z_hi});
}
inline int kernel_kind(const SphereKernel&) { return CM_SPHERE; }
inline int kernel_kind(const BoxKernel&) { return CM_CUBE; }
inline int kernel_kind(const CylinderKernel&) { return CM_CYLINDER; }

inline Csr take(cm_csr* csr) {
  std::uint64_t nq = 0, nnz = 0;
  cm_csr_info(csr, &nq, &nnz, nullptr, nullptr);
  Csr out;
  out.row_ptr.resize(nq + 1);
  out.cols.resize(nnz);
  const cm_status s = cm_csr_download(csr, out.row_ptr.data(), out.cols.data(), nullptr);
  cm_csr_free(csr);
  check(s);
  return out;
}
}  // namespace detail

// kernel_search for a batch of kernels of one type (sorted rows).
template <class K>
Csr kernel_search_batch(const Cheesemap& m, const std::vector<K>& kernels,
                        std::vector<QueryStats>* stats = nullptr) {
  std::vector<double> p;
  for (const K& k : kernels) detail::kernel_params(k, p);
  const int kind = kernels.empty() ? CM_SPHERE : detail::kernel_kind(kernels.front());
  cm_csr* csr = nullptr;
  check(cm_kernel_search(m.handle(), kind, p.data(), kernels.size(), nullptr, &csr));
  if (stats) {
    std::vector<std::uint64_t> tested(kernels.size()), voxels(kernels.size());
    const cm_status s = cm_kernel_count(m.handle(), kind, p.data(), kernels.size(), nullptr,
                                        tested.data(), voxels.data(), nullptr);
    if (s != CM_OK) cm_csr_free(csr);
    check(s);
    stats->assign(kernels.size(), QueryStats{});
    for (std::size_t q = 0; q < kernels.size(); ++q)
      (*stats)[q].points_tested = tested[q], (*stats)[q].voxels_visited = voxels[q];
  }
  return detail::take(csr);
}

// kernel_search (search.hpp:102-127): handles sorted ascending; QueryStats
// voxels_visited / points_tested equal the reference's counters.
template <class K>
std::vector<PointHandle> kernel_search(const Cheesemap& m, const K& kernel,
                                       QueryStats* stats = nullptr) {
  std::vector<QueryStats> st;
  const Csr c = kernel_search_batch(m, std::vector<K>{kernel}, stats ? &st : nullptr);
  if (stats) *stats = st[0];
  return {c.cols.begin(), c.cols.end()};
}

// baseline.hpp:11-21: the linear-scan oracle (ascending handles).
template <class K>
std::vector<PointHandle> brute_radius(const PointCloud& cloud, const K& kernel) {
  std::vector<PointHandle> out;
  for (std::size_t h = 0; h < cloud.size(); ++h)
    if (kernel.is_inside(cloud[h])) out.push_back(h);
  return out;
}

// ---------------------------------------------------------------- io.hpp --
struct LasHeaderInfo {  // io.hpp:11-19
  std::uint8_t version_major = 0, version_minor = 0, point_format = 0;
  std::uint64_t point_count = 0;
  double scale_x = 0.0, scale_y = 0.0, scale_z = 0.0;
  double offset_x = 0.0, offset_y = 0.0, offset_z = 0.0;
  Aabb bounds;
};
struct LasFile {  // io.hpp:21-24
  PointCloud cloud;
  LasHeaderInfo header;
};

// read_las (io.hpp:39-42): header checks on the host, records decoded on
// the device; throws IoError / ParseError with the reference's messages.
inline LasFile read_las(const std::string& path, int device = 0) {
  cm_las_header h;
  check(cm_las_read(path.c_str(), nullptr, 0, &h, device, nullptr));
  LasFile f;
  f.cloud.resize(h.point_count);
  check(cm_las_read(path.c_str(), reinterpret_cast<double*>(f.cloud.data()), h.point_count, &h,
                    device, nullptr));
  LasHeaderInfo& o = f.header;
  o.version_major = h.version_major, o.version_minor = h.version_minor;
  o.point_format = h.point_format, o.point_count = h.point_count;
  o.scale_x = h.scale[0], o.scale_y = h.scale[1], o.scale_z = h.scale[2];
  o.offset_x = h.offset[0], o.offset_y = h.offset[1], o.offset_z = h.offset[2];
  o.bounds.min = {h.bounds_min[0], h.bounds_min[1], h.bounds_min[2]};
  o.bounds.max = {h.bounds_max[0], h.bounds_max[1], h.bounds_max[2]};
  return f;
}

// ---------------------------------------------------------- analysis.hpp --
struct DensityHistogram {
  std::uint64_t bins[256] = {};
};
struct WeightedDensity {
  double value = 0.0;
  DensityHistogram histogram;
};

inline double global_density(const PointCloud& cloud, int device = 0) {
  double v = 0.0;
  check(cm_global_density(reinterpret_cast<const double*>(cloud.data()), cloud.size(), device,
                          nullptr, &v));
  return v;
}

inline WeightedDensity weighted_density(const PointCloud& cloud, std::uint64_t sample_size = 0,
                                        std::uint64_t sample_seed = 0, int device = 0) {
  WeightedDensity wd;
  check(cm_weighted_density(reinterpret_cast<const double*>(cloud.data()), cloud.size(),
                            sample_size, sample_seed, device, nullptr, &wd.value,
                            wd.histogram.bins));
  return wd;
}

// (idx, d2) rows of width k, ordered by (d2, handle).
inline void knn_batch(const Cheesemap& m, const std::vector<Point3>& centers, std::size_t k,
                      std::vector<std::uint32_t>& idx, std::vector<double>& d2) {
  idx.resize(centers.size() * k);
  d2.resize(centers.size() * k);
  check(cm_knn(m.handle(), reinterpret_cast<const double*>(centers.data()), centers.size(),
               static_cast<uint32_t>(k), idx.data(), d2.data(), nullptr));
}

// knn_search (search.hpp:131-134): exact for either policy; see the header
// comment for what QueryStats reports.
inline std::vector<Neighbor> knn_search(const Cheesemap& m, const Point3& c, std::size_t k,
                                        GrowthPolicy policy = GrowthPolicy::Density,
                                        QueryStats* stats = nullptr) {
  (void)policy;
  if (k == 0) throw InvalidArgumentError("k must be at least 1");
  std::vector<std::uint32_t> idx;
  std::vector<double> d2;
  knn_batch(m, {c}, k, idx, d2);
  std::vector<Neighbor> out;
  double dk = 0.0;
  for (std::size_t t = 0; t < k; ++t)
    if (idx[t] != 0xffffffffu) {
      out.push_back({idx[t], std::sqrt(d2[t])});
      dk = d2[t];
    }
  if (stats) {
    *stats = QueryStats{};
    const double r = std::sqrt(dk);
    const double p[4] = {c.x, c.y, c.z, r};
    check(cm_kernel_count(m.handle(), CM_SPHERE, p, 1, nullptr, &stats->points_tested,
                          &stats->voxels_visited, nullptr));
    stats->final_radius = r;
  }
  return out;
}

// Per-centre (count, sum of splitmix64(handle)) for outputs too large to keep.
inline void radius_digest(const Cheesemap& m, const std::vector<Point3>& centers, double r,
                          cm_kernel kind, std::vector<std::uint32_t>& counts,
                          std::vector<std::uint64_t>& digests) {
  counts.resize(centers.size());
  digests.resize(centers.size());
  check(cm_radius_digest(m.handle(), reinterpret_cast<const double*>(centers.data()),
                         centers.size(), kind, r, counts.data(), digests.data(), nullptr));
}

}  // namespace cheesemap::gpu
