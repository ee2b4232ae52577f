// TEST INFRASTRUCTURE — CPU oracle for the cheesemap build + query path.
//
// This file is a from-scratch CPU restatement of the reference algorithm
// (/root/reference/proj/core). It exists only to CHECK the CUDA path: only
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load it.
// The product (paper_2502_11602_b200/) never links or calls it.
//
// Parity pinning: the restatement is validated against the reference itself,
// compiled from its own sources into oracle/_ref/ (see oracle/Makefile and
// oracle/refshim.cpp), and against golden vectors in tests/golden/ produced
// by that build (tests/golden/make_golden.py).
//
// Compile without -march and with -ffp-contract=off (oracle/Makefile): the
// reference's Release flags (proj/CMakeLists.txt:4-9) produce no FMA, and the
// GPU path must reproduce that arithmetic.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numbers>
#include <limits>
#include <optional>
#include <random>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

namespace {

enum Status { OK = 0, EMPTY_CLOUD = 1, INVALID_ARGUMENT = 2, CAPACITY = 3, OUT_OF_DOMAIN = 4 };

struct P3 {
  double x, y, z;
};
struct Box {
  P3 lo, hi;
};
struct Range {
  std::uint64_t lo[3], hi[3];
};

// geometry.hpp:26-31 — ((dx*dx + dy*dy) + dz*dz), dx = p - c
inline double sqdist(const P3& a, const P3& b) {
  const double dx = a.x - b.x;
  const double dy = a.y - b.y;
  const double dz = a.z - b.z;
  return dx * dx + dy * dy + dz * dz;
}

// geometry.hpp:48-51 (closed)
inline bool box_contains(const Box& b, const P3& p) {
  return p.x >= b.lo.x && p.x <= b.hi.x && p.y >= b.lo.y && p.y <= b.hi.y &&
         p.z >= b.lo.z && p.z <= b.hi.z;
}
// geometry.hpp:53-56
inline bool box_intersects(const Box& a, const Box& o) {
  return a.lo.x <= o.hi.x && a.hi.x >= o.lo.x && a.lo.y <= o.hi.y &&
         a.hi.y >= o.lo.y && a.lo.z <= o.hi.z && a.hi.z >= o.lo.z;
}

// grid.cpp:29-37
inline std::uint64_t axis_index(double coord, double origin, double cell, std::uint64_t n) {
  const double idx = std::floor((coord - origin) / cell);
  if (idx < 0.0) return 0;
  const auto u = static_cast<std::uint64_t>(idx);
  return std::min(u, n - 1);
}

struct Grid {
  P3 origin;
  double cell[3];
  std::uint64_t n[3];
  int mode3d;
  Box bounds;

  std::uint64_t total() const { return n[0] * n[1] * n[2]; }
  // grid.hpp:65-67 (k fastest)
  std::uint64_t gidx(std::uint64_t i, std::uint64_t j, std::uint64_t k) const {
    return i * (n[1] * n[2]) + j * n[2] + k;
  }
  // grid.cpp:63-72 (the bounds check cannot fire for build points)
  std::uint64_t key_of(const P3& p) const {
    const std::uint64_t i = axis_index(p.x, origin.x, cell[0], n[0]);
    const std::uint64_t j = axis_index(p.y, origin.y, cell[1], n[1]);
    const std::uint64_t k = mode3d ? axis_index(p.z, origin.z, cell[2], n[2]) : 0;
    return gidx(i, j, k);
  }
  // grid.cpp:90-114
  std::optional<Range> clamped_range(const Box& q) const {
    if (!box_intersects(q, bounds)) return std::nullopt;
    Range r;
    r.lo[0] = axis_index(std::max(q.lo.x, bounds.lo.x), origin.x, cell[0], n[0]);
    r.hi[0] = axis_index(std::min(q.hi.x, bounds.hi.x), origin.x, cell[0], n[0]);
    r.lo[1] = axis_index(std::max(q.lo.y, bounds.lo.y), origin.y, cell[1], n[1]);
    r.hi[1] = axis_index(std::min(q.hi.y, bounds.hi.y), origin.y, cell[1], n[1]);
    if (mode3d) {
      r.lo[2] = axis_index(std::max(q.lo.z, bounds.lo.z), origin.z, cell[2], n[2]);
      r.hi[2] = axis_index(std::min(q.hi.z, bounds.hi.z), origin.z, cell[2], n[2]);
    } else {
      r.lo[2] = r.hi[2] = 0;
    }
    return r;
  }
  // grid.cpp:74-88
  Box voxel_bounds(std::uint64_t i, std::uint64_t j, std::uint64_t k) const {
    Box b;
    b.lo.x = origin.x + static_cast<double>(i) * cell[0];
    b.hi.x = origin.x + static_cast<double>(i + 1) * cell[0];
    b.lo.y = origin.y + static_cast<double>(j) * cell[1];
    b.hi.y = origin.y + static_cast<double>(j + 1) * cell[1];
    if (mode3d) {
      b.lo.z = origin.z + static_cast<double>(k) * cell[2];
      b.hi.z = origin.z + static_cast<double>(k + 1) * cell[2];
    } else {
      b.lo.z = bounds.lo.z;
      b.hi.z = bounds.hi.z;
    }
    return b;
  }
};

// grid.cpp:18-27; returns status
int axis_dim(double lo, double hi, double cell, std::uint64_t* out) {
  if (!(cell > 0.0)) return INVALID_ARGUMENT;
  const double n = std::floor((hi - lo) / cell) + 1.0;
  if (n >= 9.3e18) return CAPACITY;
  *out = static_cast<std::uint64_t>(n);
  return OK;
}

}  // namespace

// One sorted (key, handle) table serves all three flavours: per-voxel handle
// sets are flavour-independent (test_map.cpp:99-127), and the handles inside
// a voxel are ascending (insertion order, map.cpp:48-49, 76-78, 84-86).
struct orc_index {
  std::vector<P3> pts;
  Grid g;
  int flavor = 0;
  double tau = 0.8;
  std::vector<std::uint64_t> keys;     // sorted, n
  std::vector<std::uint64_t> handles;  // stable order, n
  std::vector<std::uint64_t> offsets;  // dense lookup (V+1) when small
  std::unordered_map<std::uint64_t, std::pair<std::uint64_t, std::uint64_t>> table;
  std::vector<std::uint64_t> slice_non_empty;
  std::uint64_t non_empty = 0;

  // [begin, end) of voxel g in keys/handles
  inline bool voxel(std::uint64_t key, std::uint64_t* b, std::uint64_t* e) const {
    if (!offsets.empty()) {
      *b = offsets[key];
      *e = offsets[key + 1];
      return *e > *b;
    }
    auto it = table.find(key);
    if (it == table.end()) return false;
    *b = it->second.first;
    *e = it->second.second;
    return true;
  }
};

namespace {

struct Stats {
  std::uint64_t voxels = 0, tested = 0;
};

// search.hpp:102-127: visit i -> j -> k over clamped_range(kernel.box()),
// test every point of every voxel. F(handle, point) is the is_inside hook.
template <class Inside, class Emit>
void kernel_search(const orc_index& m, const Box& kbox, Inside&& inside, Emit&& emit,
                   Stats* st) {
  const auto range = m.g.clamped_range(kbox);
  if (!range) return;
  for (std::uint64_t i = range->lo[0]; i <= range->hi[0]; ++i)
    for (std::uint64_t j = range->lo[1]; j <= range->hi[1]; ++j)
      for (std::uint64_t k = range->lo[2]; k <= range->hi[2]; ++k) {
        ++st->voxels;
        std::uint64_t b, e;
        if (!m.voxel(m.g.gidx(i, j, k), &b, &e)) continue;
        for (std::uint64_t p = b; p < e; ++p) {
          ++st->tested;
          const std::uint64_t h = m.handles[p];
          if (inside(m.pts[h])) emit(h);
        }
      }
}

// SphereKernel::box (geometry.hpp:77-80) / BoxKernel{c-r, c+r}
// (cmd_bench.cpp:107-111, test_search.cpp:177): the same box for both.
inline Box radius_box(const P3& c, double r) {
  return {{c.x - r, c.y - r, c.z - r}, {c.x + r, c.y + r, c.z + r}};
}

// CylinderKernel{c.x, c.y, r} with the default unbounded z range
// (geometry.hpp:97-113): box (c.x +- r, c.y +- r, -inf..inf), member iff
// z in range && squared_distance_xy <= r*r (geometry.hpp:39-43).
inline Box cylinder_box(const P3& c, double r) {
  const double inf = std::numeric_limits<double>::infinity();
  return {{c.x - r, c.y - r, -inf}, {c.x + r, c.y + r, inf}};
}
inline bool in_cylinder(const P3& p, const P3& c, double rr) {
  const double inf = std::numeric_limits<double>::infinity();
  const double dx = p.x - c.x;
  const double dy = p.y - c.y;
  return p.z >= -inf && p.z <= inf && dx * dx + dy * dy <= rr;
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

// search.cpp:9-36 — bounded list sorted by sqrt distance, ties in insertion
// order (upper_bound), overflow dropped.
struct CandidateList {
  std::size_t cap;
  std::vector<std::pair<double, std::uint64_t>> items;  // (distance, handle)
  explicit CandidateList(std::size_t c) : cap(c) { items.reserve(c + 1); }
  void insert(std::uint64_t h, double d) {
    if (items.size() == cap && d >= items.back().first) return;
    auto pos = std::upper_bound(items.begin(), items.end(), d,
                                [](double v, const auto& it) { return v < it.first; });
    items.insert(pos, {d, h});
    if (items.size() > cap) items.pop_back();
  }
  std::size_t count_within(double r) const {
    auto pos = std::upper_bound(items.begin(), items.end(), r,
                                [](double v, const auto& it) { return v < it.first; });
    return static_cast<std::size_t>(pos - items.begin());
  }
};

// search.cpp:78-83
double distance_to_box(const P3& p, const Box& b) {
  const double dx = std::max({b.lo.x - p.x, 0.0, p.x - b.hi.x});
  const double dy = std::max({b.lo.y - p.y, 0.0, p.y - b.hi.y});
  const double dz = std::max({b.lo.z - p.z, 0.0, p.z - b.hi.z});
  return std::sqrt(dx * dx + dy * dy + dz * dz);
}

// search.cpp:87-146 (Alg. 2, density growth). Returns the handles found.
std::vector<std::uint64_t> knn_alg2(const orc_index& m, const P3& c, std::size_t k,
                                    Stats* st) {
  const Grid& g = m.g;
  double step = std::max(g.cell[0], g.cell[1]);
  if (g.mode3d) step = std::max(step, g.cell[2]);
  double r;
  if (box_contains(g.bounds, c)) {
    // initial_radius, search.cpp:47-56
    const std::uint64_t i = axis_index(c.x, g.origin.x, g.cell[0], g.n[0]);
    const std::uint64_t j = axis_index(c.y, g.origin.y, g.cell[1], g.n[1]);
    const std::uint64_t kk = g.mode3d ? axis_index(c.z, g.origin.z, g.cell[2], g.n[2]) : 0;
    const Box b = g.voxel_bounds(i, j, kk);
    r = std::min(std::abs(c.x - b.lo.x), std::abs(c.x - b.hi.x));
    r = std::min(r, std::min(std::abs(c.y - b.lo.y), std::abs(c.y - b.hi.y)));
    if (g.mode3d) r = std::min(r, std::min(std::abs(c.z - b.lo.z), std::abs(c.z - b.hi.z)));
  } else {
    r = distance_to_box(c, g.bounds) + step;
  }
  CandidateList cand(k);
  std::optional<Range> taboo;
  std::optional<double> prev_density;
  for (;;) {
    const auto range = g.clamped_range(radius_box(c, r));
    if (range) {
      Range next = *range;
      if (taboo) {  // hull, grid.cpp:9-14
        for (int a = 0; a < 3; ++a) {
          next.lo[a] = std::min(next.lo[a], taboo->lo[a]);
          next.hi[a] = std::max(next.hi[a], taboo->hi[a]);
        }
      }
      // for_each_frontier_voxel, search.hpp:63-79
      for (std::uint64_t i = next.lo[0]; i <= next.hi[0]; ++i)
        for (std::uint64_t j = next.lo[1]; j <= next.hi[1]; ++j)
          for (std::uint64_t kk = next.lo[2]; kk <= next.hi[2]; ++kk) {
            if (taboo && i >= taboo->lo[0] && i <= taboo->hi[0] && j >= taboo->lo[1] &&
                j <= taboo->hi[1] && kk >= taboo->lo[2] && kk <= taboo->hi[2]) {
              kk = taboo->hi[2];
              continue;
            }
            ++st->voxels;
            std::uint64_t b, e;
            if (!m.voxel(g.gidx(i, j, kk), &b, &e)) continue;
            for (std::uint64_t p = b; p < e; ++p) {
              ++st->tested;
              const std::uint64_t h = m.handles[p];
              cand.insert(h, std::sqrt(sqdist(m.pts[h], c)));
            }
          }
      taboo = next;
    }
    const std::size_t in_ball = cand.count_within(r);
    const bool covers = taboo && taboo->lo[0] == 0 && taboo->lo[1] == 0 && taboo->lo[2] == 0 &&
                        taboo->hi[0] == g.n[0] - 1 && taboo->hi[1] == g.n[1] - 1 &&
                        taboo->hi[2] == g.n[2] - 1;
    if (in_ball >= k || covers) break;
    // grow_radius, search.cpp:58-74
    if (in_ball == 0 || r <= 0.0) {
      r = r + step;
    } else {
      const double volume = (4.0 / 3.0) * std::numbers::pi * r * r * r;
      const double density = static_cast<double>(in_ball) / volume;
      if (prev_density && density == *prev_density) {
        r = r + step;
      } else {
        const double estimate = std::cbrt(static_cast<double>(k) / density);
        r = estimate <= r ? r + step : estimate;
      }
      prev_density = density;
    }
  }
  std::vector<std::uint64_t> out;
  for (auto& it : cand.items) out.push_back(it.second);
  return out;
}

}  // namespace

extern "C" {

// Cheesemap::build (map.cpp:22-122): same checks in the same order.
static int build_impl(const double* xyz, uint64_t n, int flavor, int mode, double cx, double cy,
                      double cz, double tau, uint64_t dense_cap, const double* b6,
                      orc_index** out) {
  *out = nullptr;
  if (n == 0) return EMPTY_CLOUD;                                  // map.cpp:23-25
  if (!(tau > 0.0) || tau > 1.0) return INVALID_ARGUMENT;          // map.cpp:26-28
  auto m = new orc_index();
  m->pts.resize(n);
  std::memcpy(m->pts.data(), xyz, n * sizeof(P3));
  // aabb_of_points, geometry.cpp:7-21
  Box bb{m->pts[0], m->pts[0]};
  for (const P3& p : m->pts) {
    bb.lo.x = std::min(bb.lo.x, p.x);
    bb.lo.y = std::min(bb.lo.y, p.y);
    bb.lo.z = std::min(bb.lo.z, p.z);
    bb.hi.x = std::max(bb.hi.x, p.x);
    bb.hi.y = std::max(bb.hi.y, p.y);
    bb.hi.z = std::max(bb.hi.z, p.z);
  }
  if (b6) {  // explicit grid box; points outside it: voxel_of (grid.cpp:64-66)
    const Box eb{{b6[0], b6[1], b6[2]}, {b6[3], b6[4], b6[5]}};
    if (!box_contains(eb, bb.lo) || !box_contains(eb, bb.hi)) {
      delete m;
      return OUT_OF_DOMAIN;
    }
    bb = eb;
  }
  // grid_dims, grid.cpp:41-61
  Grid& g = m->g;
  g.origin = bb.lo;
  g.bounds = bb;
  g.cell[0] = cx;
  g.cell[1] = cy;
  g.cell[2] = cz;
  g.mode3d = mode != 0;
  int s;
  if ((s = axis_dim(bb.lo.x, bb.hi.x, cx, &g.n[0])) ||
      (s = axis_dim(bb.lo.y, bb.hi.y, cy, &g.n[1]))) {
    delete m;
    return s;
  }
  if (g.mode3d) {
    if ((s = axis_dim(bb.lo.z, bb.hi.z, cz, &g.n[2]))) {
      delete m;
      return s;
    }
  } else {
    g.n[2] = 1;
  }
  const std::uint64_t limit = std::uint64_t{1} << 63;
  if ((g.n[1] != 0 && g.n[0] > limit / g.n[1]) ||
      (g.n[2] != 0 && g.n[0] * g.n[1] > limit / g.n[2])) {
    delete m;
    return CAPACITY;
  }
  const std::uint64_t V = g.total();
  if (flavor == 0 && V > dense_cap) {  // map.cpp:35-39
    delete m;
    return CAPACITY;
  }
  m->flavor = flavor;
  m->tau = tau;
  // per-point key (map.cpp:42-45) and stable sort by key (map.cpp:51-54)
  std::vector<std::uint64_t> key(n);
  for (std::uint64_t h = 0; h < n; ++h) key[h] = g.key_of(m->pts[h]);
  m->handles.resize(n);
  for (std::uint64_t h = 0; h < n; ++h) m->handles[h] = h;
  std::stable_sort(m->handles.begin(), m->handles.end(),
                   [&](std::uint64_t a, std::uint64_t b) { return key[a] < key[b]; });
  m->keys.resize(n);
  for (std::uint64_t p = 0; p < n; ++p) m->keys[p] = key[m->handles[p]];
  const bool small = V <= 8 * n + 1024;
  if (small) m->offsets.assign(V + 1, 0);
  if (g.mode3d || true) m->slice_non_empty.assign(g.n[2], 0);
  for (std::uint64_t p = 0; p < n;) {
    std::uint64_t e = p;
    while (e < n && m->keys[e] == m->keys[p]) ++e;
    ++m->non_empty;
    ++m->slice_non_empty[m->keys[p] % g.n[2]];
    if (small) m->offsets[m->keys[p] + 1] = e - p;
    else m->table.emplace(m->keys[p], std::make_pair(p, e));
    p = e;
  }
  if (small)
    for (std::uint64_t v = 0; v < V; ++v) m->offsets[v + 1] += m->offsets[v];
  *out = m;
  return OK;
}

int orc_build(const double* xyz, uint64_t n, int flavor, int mode, double cx, double cy,
              double cz, double tau, uint64_t dense_cap, orc_index** out) {
  return build_impl(xyz, n, flavor, mode, cx, cy, cz, tau, dense_cap, nullptr, out);
}

int orc_build_in_bounds(const double* xyz, uint64_t n, int flavor, int mode, double cx, double cy,
                        double cz, double tau, uint64_t dense_cap, const double* bounds6,
                        orc_index** out) {
  return build_impl(xyz, n, flavor, mode, cx, cy, cz, tau, dense_cap, bounds6, out);
}

void orc_free(orc_index* m) { delete m; }

void orc_grid(const orc_index* m, double* origin3, double* cell3, uint64_t* dims3,
              double* bmin3, double* bmax3) {
  const Grid& g = m->g;
  origin3[0] = g.origin.x, origin3[1] = g.origin.y, origin3[2] = g.origin.z;
  for (int a = 0; a < 3; ++a) cell3[a] = g.cell[a], dims3[a] = g.n[a];
  bmin3[0] = g.bounds.lo.x, bmin3[1] = g.bounds.lo.y, bmin3[2] = g.bounds.lo.z;
  bmax3[0] = g.bounds.hi.x, bmax3[1] = g.bounds.hi.y, bmax3[2] = g.bounds.hi.z;
}

uint64_t orc_non_empty(const orc_index* m) { return m->non_empty; }

// occupancy_stats().slices for the mixed flavour (map.cpp:150-171): slice k
// densifies iff (double)non_empty / (double)(nx*ny) >= tau (map.cpp:106-108);
// non_empty only grows, so the final flag is the test on the final count.
uint64_t orc_slice_flags(const orc_index* m, uint8_t* dense, uint64_t* non_empty) {
  if (m->flavor != 2) return 0;  // slices are reported for the mixed flavour only
  const double fp = static_cast<double>(m->g.n[0] * m->g.n[1]);
  for (std::uint64_t k = 0; k < m->slice_non_empty.size(); ++k) {
    if (non_empty) non_empty[k] = m->slice_non_empty[k];
    if (dense) dense[k] = static_cast<double>(m->slice_non_empty[k]) / fp >= m->tau;
  }
  return m->slice_non_empty.size();
}

// memory_report (map.cpp:173-192) with the cost model of map.cpp:14-18:
// out3 = {handle_bytes, structure_bytes, total_bytes}.
void orc_memory_report(const orc_index* m, uint64_t* out3) {
  const std::uint64_t V = m->g.n[0] * m->g.n[1] * m->g.n[2];
  const std::uint64_t hb = 8 * m->pts.size();
  std::uint64_t sb = 0;
  if (m->flavor == 0) {
    sb = 8 * (V + 1);
  } else if (m->flavor == 1) {
    sb = 64 * m->non_empty;
  } else {
    const std::uint64_t fp = m->g.n[0] * m->g.n[1];
    for (const std::uint64_t ne : m->slice_non_empty) {
      const bool dense = static_cast<double>(ne) / static_cast<double>(fp) >= m->tau;
      sb += 48 + (dense ? 24 * fp : 64 * ne);
    }
  }
  out3[0] = hb;
  out3[1] = sb;
  out3[2] = hb + sb;
}

// (key, handle) in stored order: key ascending, handles ascending per voxel.
void orc_export(const orc_index* m, uint64_t* keys, uint64_t* handles) {
  const std::uint64_t n = m->keys.size();
  if (keys) std::memcpy(keys, m->keys.data(), n * 8);
  if (handles) std::memcpy(handles, m->handles.data(), n * 8);
}

uint64_t orc_mix64(uint64_t x) { return mix64(x); }

// Batched kernel_search (search.hpp:102-127) with kernel 0 = SphereKernel
// (geometry.hpp:73-85), 1 = BoxKernel{c-r, c+r} (geometry.hpp:87-92).
// Per query: neighbour count, set digest sum(mix64(handle)) mod 2^64, and the
// reference's QueryStats counters (search.hpp:12-17). Any output may be null.
int orc_radius(const orc_index* m, const double* q, uint64_t nq, int kernel, double r,
               unsigned threads, uint32_t* counts, uint64_t* digests,
               uint64_t* points_tested, uint64_t* voxels_visited) {
  if (kernel < 0 || kernel > 2) return INVALID_ARGUMENT;
  const double rr = r * r;
  parallel_queries(nq, threads, [&](std::uint64_t qi) {
    const P3 c{q[3 * qi], q[3 * qi + 1], q[3 * qi + 2]};
    const Box kb = radius_box(c, r);
    Stats st;
    std::uint64_t cnt = 0, dig = 0;
    auto emit = [&](std::uint64_t h) {
      ++cnt;
      dig += mix64(h);
    };
    if (kernel == 0)
      kernel_search(*m, kb, [&](const P3& p) { return sqdist(p, c) <= rr; }, emit, &st);
    else if (kernel == 1)
      kernel_search(*m, kb, [&](const P3& p) { return box_contains(kb, p); }, emit, &st);
    else
      kernel_search(*m, cylinder_box(c, r), [&](const P3& p) { return in_cylinder(p, c, rr); },
                    emit, &st);
    if (counts) counts[qi] = static_cast<uint32_t>(cnt);
    if (digests) digests[qi] = dig;
    if (points_tested) points_tested[qi] = st.tested;
    if (voxels_visited) voxels_visited[qi] = st.voxels;
  });
  return OK;
}

// Sorted neighbour lists (the reference tests sort kernel_search output:
// tests/test_util.hpp:30-35) written at row_ptr[q] (row_ptr from the counts).
int orc_radius_fill(const orc_index* m, const double* q, uint64_t nq, int kernel, double r,
                    unsigned threads, const uint64_t* row_ptr, uint32_t* cols) {
  if (kernel < 0 || kernel > 2) return INVALID_ARGUMENT;
  const double rr = r * r;
  parallel_queries(nq, threads, [&](std::uint64_t qi) {
    const P3 c{q[3 * qi], q[3 * qi + 1], q[3 * qi + 2]};
    const Box kb = radius_box(c, r);
    Stats st;
    std::vector<std::uint32_t> hits;
    auto emit = [&](std::uint64_t h) { hits.push_back(static_cast<uint32_t>(h)); };
    if (kernel == 0)
      kernel_search(*m, kb, [&](const P3& p) { return sqdist(p, c) <= rr; }, emit, &st);
    else if (kernel == 1)
      kernel_search(*m, kb, [&](const P3& p) { return box_contains(kb, p); }, emit, &st);
    else
      kernel_search(*m, cylinder_box(c, r), [&](const P3& p) { return in_cylinder(p, c, rr); },
                    emit, &st);
    std::sort(hits.begin(), hits.end());
    std::copy(hits.begin(), hits.end(), cols + row_ptr[qi]);
  });
  return OK;
}

// kNN restatement: run Alg. 2 (search.cpp:87-146) to get a
// set of k handles; D = max d^2 over them; a custom kernel
// {d^2 <= D} through kernel_search (the reference's Kernel extension point,
// geometry.hpp:67-71) collects every point at d^2 <= D; sort by (d^2, handle)
// and keep k. Output rows are k wide; missing entries (k > N) are
// UINT32_MAX / +inf. points_tested_rk: candidates of kernel_search with the
// exact k-th distance (the roofline byte basis).
int orc_knn(const orc_index* m, const double* q, uint64_t nq, uint32_t k, unsigned threads,
            uint32_t* idx_out, double* d2_out, uint64_t* points_tested_rk,
            uint64_t* points_tested_alg2) {
  if (k == 0) return INVALID_ARGUMENT;  // search.cpp:90-92
  parallel_queries(nq, threads, [&](std::uint64_t qi) {
    const P3 c{q[3 * qi], q[3 * qi + 1], q[3 * qi + 2]};
    Stats st;
    const auto found = knn_alg2(*m, c, k, &st);
    if (points_tested_alg2) points_tested_alg2[qi] = st.tested;
    double D = 0.0;
    for (std::uint64_t h : found) D = std::max(D, sqdist(m->pts[h], c));
    const double rb = std::sqrt(D) * (1.0 + 1e-9) + 1e-300;
    std::vector<std::pair<double, std::uint64_t>> all;
    Stats st2;
    kernel_search(*m, radius_box(c, rb), [&](const P3& p) { return sqdist(p, c) <= D; },
                  [&](std::uint64_t h) { all.push_back({sqdist(m->pts[h], c), h}); }, &st2);
    std::sort(all.begin(), all.end());
    for (uint32_t t = 0; t < k; ++t) {
      if (t < all.size()) {
        idx_out[qi * k + t] = static_cast<uint32_t>(all[t].second);
        if (d2_out) d2_out[qi * k + t] = all[t].first;
      } else {
        idx_out[qi * k + t] = UINT32_MAX;
        if (d2_out) d2_out[qi * k + t] = INFINITY;
      }
    }
    if (points_tested_rk) {
      // candidates of a sphere query at the exact k-th distance
      const double dk = all.empty() ? 0.0 : std::sqrt(all[std::min<std::size_t>(k, all.size()) - 1].first);
      Stats st3;
      kernel_search(*m, radius_box(c, dk), [](const P3&) { return false; },
                    [](std::uint64_t) {}, &st3);
      points_tested_rk[qi] = st3.tested;
    }
  });
  return OK;
}

// weighted_density (analysis.cpp:26-86): optional seeded subsample (partial
// Fisher-Yates with mt19937_64, :36-45), a 2D sparse map at 1 m, per sampled
// point the count of points in a vertical 1 m cylinder, local density
// count / pi floored into 256 bins (last bin clamps), value = histogram-
// weighted mean of the bin indices.
int orc_weighted_density(const double* xyz, uint64_t n, uint64_t sample_size, uint64_t seed,
                         unsigned threads, double* value, uint64_t* bins256) {
  if (n == 0) return EMPTY_CLOUD;
  std::vector<std::uint64_t> sample;
  if (sample_size && sample_size < n) {
    sample.resize(n);
    for (std::uint64_t i = 0; i < n; ++i) sample[i] = i;
    std::mt19937_64 eng(seed);
    for (std::uint64_t i = 0; i < sample_size; ++i) {
      const std::uint64_t j = i + eng() % (sample.size() - i);
      std::swap(sample[i], sample[j]);
    }
    sample.resize(sample_size);
  } else {
    sample.resize(n);
    for (std::uint64_t i = 0; i < n; ++i) sample[i] = i;
  }
  orc_index* m = nullptr;
  int s = orc_build(xyz, n, 1, 0, 1.0, 1.0, 1.0, 0.8, 1ull << 32, &m);
  if (s) return s;
  std::vector<double> q(3 * sample.size());
  for (std::size_t i = 0; i < sample.size(); ++i)
    for (int a = 0; a < 3; ++a) q[3 * i + a] = xyz[3 * sample[i] + a];
  std::vector<uint32_t> counts(sample.size());
  orc_radius(m, q.data(), sample.size(), 2, 1.0, threads, counts.data(), nullptr, nullptr, nullptr);
  orc_free(m);
  for (int b = 0; b < 256; ++b) bins256[b] = 0;
  for (uint32_t c : counts) {
    const double local = static_cast<double>(c) / std::numbers::pi;
    const auto bin = std::min<std::uint64_t>(255, static_cast<std::uint64_t>(local));
    ++bins256[bin];
  }
  std::uint64_t ws = 0, tot = 0;
  for (int b = 0; b < 256; ++b) {
    ws += b * bins256[b];
    tot += bins256[b];
  }
  *value = static_cast<double>(ws) / static_cast<double>(tot);
  return OK;
}

// ---- read_las restated (io.cpp:33-106) over an in-memory image ------------
// Same checks, messages and order as the reference; coordinate =
// raw * scale + offset (int32 promoted to double, no FMA: -ffp-contract=off).
// Status: 0 ok, 7 ParseError, 2 capacity too small. `msg` gets the message.
struct orc_las_header {
  uint8_t version_major, version_minor, point_format;
  uint16_t header_size, record_length;
  uint32_t data_offset;
  uint64_t point_count;
  double scale[3], offset[3];
  double bounds_min[3], bounds_max[3];
};

static int las_fail(char* msg, int msglen, const std::string& m, int code) {
  if (msg && msglen > 0) {
    std::strncpy(msg, m.c_str(), (size_t)msglen - 1);
    msg[msglen - 1] = 0;
  }
  return code;
}

extern "C++" {
template <class T>
static T las_rd(const unsigned char* b, size_t off) {
  T v;
  std::memcpy(&v, b + off, sizeof(T));
  return v;
}
}

int orc_las_read(const void* bytes, uint64_t n, const char* name, orc_las_header* h,
                 double* xyz, uint64_t cap, char* msg, int msglen) {
  const unsigned char* b = static_cast<const unsigned char*>(bytes);
  const std::string nm = name ? name : "";
  if (n < 227 || std::memcmp(b, "LASF", 4) != 0)  // io.cpp:44-47
    return las_fail(msg, msglen, "bad LAS magic at byte 0 in " + nm, 7);
  std::memset(h, 0, sizeof(*h));
  h->version_major = b[24];  // io.cpp:49-56
  h->version_minor = b[25];
  if (h->version_major != 1 || h->version_minor < 2 || h->version_minor > 4)
    return las_fail(msg, msglen,
                    "unsupported LAS version " + std::to_string(h->version_major) + "." +
                        std::to_string(h->version_minor), 7);
  h->header_size = las_rd<uint16_t>(b, 94);  // io.cpp:57-62
  h->data_offset = las_rd<uint32_t>(b, 96);
  h->point_format = b[104];
  if (h->point_format > 8)
    return las_fail(msg, msglen,
                    "unsupported LAS point record format " + std::to_string(h->point_format), 7);
  h->record_length = las_rd<uint16_t>(b, 105);  // io.cpp:63-67
  if (h->record_length < 12)
    return las_fail(msg, msglen,
                    "LAS point record length " + std::to_string(h->record_length) +
                        " is too short", 7);
  h->point_count = las_rd<uint32_t>(b, 107);  // io.cpp:68-71
  if (h->point_count == 0 && h->version_minor == 4 && h->header_size >= 255)
    h->point_count = n >= 255 ? las_rd<uint64_t>(b, 247) : 0;
  for (int a = 0; a < 3; ++a) h->scale[a] = las_rd<double>(b, 131 + 8 * a);  // io.cpp:72-77
  if (!(h->scale[0] > 0.0) || !(h->scale[1] > 0.0) || !(h->scale[2] > 0.0))
    return las_fail(msg, msglen, "non-positive LAS scale factor at byte 131", 7);
  for (int a = 0; a < 3; ++a) h->offset[a] = las_rd<double>(b, 155 + 8 * a);  // io.cpp:78-86
  for (int a = 0; a < 3; ++a) {
    h->bounds_max[a] = las_rd<double>(b, 179 + 16 * a);
    h->bounds_min[a] = las_rd<double>(b, 187 + 16 * a);
  }
  if (h->data_offset < h->header_size || h->data_offset > n)  // io.cpp:88-91
    return las_fail(msg, msglen,
                    "LAS point data offset " + std::to_string(h->data_offset) +
                        " is out of range", 7);
  if (!xyz) return 0;
  uint64_t pos = h->data_offset;
  for (uint64_t i = 0; i < h->point_count; ++i, pos += h->record_length) {  // io.cpp:93-105
    if (pos + h->record_length > n)
      return las_fail(msg, msglen,
                      "truncated LAS point record " + std::to_string(i) + " at byte " +
                          std::to_string(pos), 7);
    if (i >= cap) return las_fail(msg, msglen, "capacity", 2);
    const int32_t rx = las_rd<int32_t>(b, pos), ry = las_rd<int32_t>(b, pos + 4),
                  rz = las_rd<int32_t>(b, pos + 8);
    xyz[3 * i] = rx * h->scale[0] + h->offset[0];
    xyz[3 * i + 1] = ry * h->scale[1] + h->offset[1];
    xyz[3 * i + 2] = rz * h->scale[2] + h->offset[2];
  }
  return 0;
}

}  // extern "C"
