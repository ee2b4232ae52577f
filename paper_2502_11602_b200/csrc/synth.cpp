// Seeded synthetic LiDAR clouds for the BASELINE.json configs (host C++).
//
// The reference ships only uniform-box / void-ellipse / gaussian-cluster
// generators (proj/core/src/io.cpp:252-335); none of the BASELINE configs
// (ALS terrain + vegetation + buildings, TLS scanner) exist there. These
// generators reuse the reference's RNG bit conventions:
//   * std::mt19937_64(seed),
//   * uniform01 = (eng() >> 11) * 2^-53, uniform(lo,hi) = lo + (hi-lo)*u
//     (io.cpp:221-227),
//   * splitmix64 query-centre stream (tools/common.cpp:109-125).
// Every decision the BASELINE leaves open is fixed here and recorded in
// DESIGN.md §"Synthetic inputs".
//
// Determinism: the ALS ground layer is generated in fixed-size chunks, each
// with its own mt19937_64 seeded from (seed, chunk), and every TLS ray draws
// its range noise from a counter-based splitmix64 stream, so the output is
// bit-identical for any host thread count.
//
// Compiled with -ffp-contract=off: coordinates must not depend on whether
// the host compiler contracts a*b+c.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numbers>
#include <random>
#include <thread>
#include <vector>

namespace {

constexpr double kTwoPi = 2.0 * std::numbers::pi;

std::uint64_t mix64(std::uint64_t x) {  // splitmix64 finaliser
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

class Rng {  // io.cpp:217-248 conventions
 public:
  explicit Rng(std::uint64_t seed) : eng_(seed) {}
  double uniform01() { return static_cast<double>(eng_() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform01(); }
  std::uint64_t index(std::uint64_t n) { return eng_() % n; }
  // Box-Muller with the cached second value (io.cpp:231-243)
  double gaussian(double mean, double sigma) {
    if (has_spare_) {
      has_spare_ = false;
      return mean + sigma * spare_;
    }
    const double u1 = static_cast<double>((eng_() >> 11) + 1) * 0x1.0p-53;  // (0, 1]
    const double u2 = uniform01();
    const double mag = std::sqrt(-2.0 * std::log(u1));
    spare_ = mag * std::sin(2.0 * std::numbers::pi * u2);
    has_spare_ = true;
    return mean + sigma * mag * std::cos(2.0 * std::numbers::pi * u2);
  }

 private:
  std::mt19937_64 eng_;
  bool has_spare_ = false;
  double spare_ = 0.0;
};

unsigned worker_count(unsigned requested) {
  if (requested > 0) return requested;
  unsigned hc = std::thread::hardware_concurrency();
  return hc == 0 ? 1u : hc;
}

template <class F>
void parallel_for(std::uint64_t n, unsigned threads, F&& f) {
  threads = static_cast<unsigned>(std::min<std::uint64_t>(threads, std::max<std::uint64_t>(n, 1)));
  if (threads <= 1) {
    for (std::uint64_t i = 0; i < n; ++i) f(i);
    return;
  }
  std::atomic<std::uint64_t> next{0};
  std::vector<std::thread> pool;
  for (unsigned t = 0; t < threads; ++t) {
    pool.emplace_back([&] {
      for (;;) {
        const std::uint64_t i = next.fetch_add(1);
        if (i >= n) return;
        f(i);
      }
    });
  }
  for (auto& th : pool) th.join();
}

// ---------------------------------------------------------------- ALS ----

struct Wave {
  double fx, fy, phase;
};

struct Building {
  double x0, x1, y0, y1, z0, z1;
  std::uint64_t points;  // surface samples (roof + 4 walls)
};

struct AlsModel {
  Wave waves[4];
  std::vector<Building> buildings;
  double ex, ey;
  double density;  // points per m^2 of the full square
};

// z = sum of 4 random-phase sinusoids, 2.5 m each (10 m total amplitude).
double terrain(const AlsModel& m, double x, double y) {
  double z = 0.0;
  for (const Wave& w : m.waves) {
    z = z + 2.5 * std::sin(kTwoPi * (w.fx * x + w.fy * y) + w.phase);
  }
  return z;
}

AlsModel make_als_model(std::uint64_t seed, std::uint64_t n, double ex,
                        double ey, std::uint32_t n_buildings) {
  AlsModel m;
  m.ex = ex;
  m.ey = ey;
  m.density = static_cast<double>(n) / (ex * ey);
  Rng rng(seed);
  for (Wave& w : m.waves) {
    const double lambda = rng.uniform(50.0, 250.0);
    const double theta = rng.uniform(0.0, kTwoPi);
    w.fx = std::cos(theta) / lambda;
    w.fy = std::sin(theta) / lambda;
    w.phase = rng.uniform(0.0, kTwoPi);
  }
  for (std::uint32_t b = 0; b < n_buildings; ++b) {
    const double sx = rng.uniform(10.0, 40.0);
    const double sy = rng.uniform(10.0, 40.0);
    const double h = rng.uniform(5.0, 30.0);
    const double cx = rng.uniform(sx / 2.0, ex - sx / 2.0);
    const double cy = rng.uniform(sy / 2.0, ey - sy / 2.0);
    Building bd;
    bd.x0 = cx - sx / 2.0;
    bd.x1 = cx + sx / 2.0;
    bd.y0 = cy - sy / 2.0;
    bd.y1 = cy + sy / 2.0;
    bd.z0 = terrain(m, cx, cy);
    bd.z1 = bd.z0 + h;
    const double area = sx * sy + 2.0 * h * (sx + sy);
    bd.points = static_cast<std::uint64_t>(std::llround(area * m.density));
    m.buildings.push_back(bd);
  }
  return m;
}

constexpr std::uint64_t kChunk = 1u << 16;

// Coarse 10 m bucket index of building footprints for ground rejection.
struct FootprintIndex {
  double cell = 10.0;
  std::uint64_t nx = 0, ny = 0;
  std::vector<std::vector<std::uint32_t>> buckets;

  FootprintIndex(const AlsModel& m) {
    nx = static_cast<std::uint64_t>(m.ex / cell) + 1;
    ny = static_cast<std::uint64_t>(m.ey / cell) + 1;
    buckets.resize(nx * ny);
    for (std::uint32_t b = 0; b < m.buildings.size(); ++b) {
      const Building& bd = m.buildings[b];
      const auto i0 = static_cast<std::uint64_t>(std::max(0.0, bd.x0 / cell));
      const auto i1 = std::min<std::uint64_t>(nx - 1, static_cast<std::uint64_t>(bd.x1 / cell));
      const auto j0 = static_cast<std::uint64_t>(std::max(0.0, bd.y0 / cell));
      const auto j1 = std::min<std::uint64_t>(ny - 1, static_cast<std::uint64_t>(bd.y1 / cell));
      for (std::uint64_t i = i0; i <= i1; ++i)
        for (std::uint64_t j = j0; j <= j1; ++j) buckets[i * ny + j].push_back(b);
    }
  }

  bool covered(const AlsModel& m, double x, double y) const {
    const auto i = std::min<std::uint64_t>(nx - 1, static_cast<std::uint64_t>(x / cell));
    const auto j = std::min<std::uint64_t>(ny - 1, static_cast<std::uint64_t>(y / cell));
    for (std::uint32_t b : buckets[i * ny + j]) {
      const Building& bd = m.buildings[b];
      if (x >= bd.x0 && x <= bd.x1 && y >= bd.y0 && y <= bd.y1) return true;
    }
    return false;
  }
};

void sample_building(const Building& bd, std::uint64_t seed, std::uint64_t b,
                     double* out) {
  Rng rng(mix64(seed ^ mix64(0x100000000ull + b)));
  const double sx = bd.x1 - bd.x0, sy = bd.y1 - bd.y0, h = bd.z1 - bd.z0;
  const double roof = sx * sy, wall_x = sx * h, wall_y = sy * h;
  const double total = roof + 2.0 * wall_x + 2.0 * wall_y;
  for (std::uint64_t p = 0; p < bd.points; ++p) {
    const double face = rng.uniform01() * total;
    const double u = rng.uniform01();
    const double v = rng.uniform01();
    double x, y, z;
    if (face < roof) {
      x = bd.x0 + sx * u;
      y = bd.y0 + sy * v;
      z = bd.z1;
    } else if (face < roof + wall_x) {
      x = bd.x0 + sx * u;
      y = bd.y0;
      z = bd.z0 + h * v;
    } else if (face < roof + 2.0 * wall_x) {
      x = bd.x0 + sx * u;
      y = bd.y1;
      z = bd.z0 + h * v;
    } else if (face < roof + 2.0 * wall_x + wall_y) {
      x = bd.x0;
      y = bd.y0 + sy * u;
      z = bd.z0 + h * v;
    } else {
      x = bd.x1;
      y = bd.y0 + sy * u;
      z = bd.z0 + h * v;
    }
    out[3 * p + 0] = x;
    out[3 * p + 1] = y;
    out[3 * p + 2] = z;
  }
}

}  // namespace

extern "C" {

uint64_t cms_mix64(uint64_t x) { return mix64(x); }

// Number of building-surface points the ALS generator will emit (so callers
// can report the ground/building split). Building points are taken out of
// the n-point budget; returns UINT64_MAX if they would exceed it.
uint64_t cms_als_building_points(uint64_t seed, uint64_t n, double ex, double ey,
                                 uint32_t n_buildings) {
  const AlsModel m = make_als_model(seed, n, ex, ey, n_buildings);
  std::uint64_t total = 0;
  for (const Building& b : m.buildings) total += b.points;
  return total > n ? UINT64_MAX : total;
}

// ALS-like tile: n points over [0,ex)x[0,ey); terrain of 4 sinusoids
// (2.5 m each, wavelength U[50,250] m, direction U[0,2pi), phase U[0,2pi));
// 30% of ground samples lifted by U(0,20) m (vegetation); n_buildings
// axis-aligned boxes (sides U[10,40] m, height U[5,30] m, base on the
// terrain at the box centre) whose roof and walls are sampled at the
// cloud's mean density. Ground samples inside a footprint are rejected.
// Output order: ground chunks, then buildings. Returns 0 on success.
int cms_generate_als(uint64_t seed, uint64_t n, double ex, double ey,
                     uint32_t n_buildings, uint32_t threads, double* xyz) {
  if (n == 0 || !(ex > 0.0) || !(ey > 0.0) || xyz == nullptr) return 2;
  const AlsModel m = make_als_model(seed, n, ex, ey, n_buildings);
  std::uint64_t bpts = 0;
  for (const Building& b : m.buildings) bpts += b.points;
  if (bpts > n) return 2;
  const std::uint64_t n_ground = n - bpts;
  const FootprintIndex fp(m);
  const unsigned T = worker_count(threads);

  const std::uint64_t chunks = (n_ground + kChunk - 1) / kChunk;
  parallel_for(chunks, T, [&](std::uint64_t c) {
    Rng rng(mix64(seed ^ mix64(c + 1)));
    const std::uint64_t begin = c * kChunk;
    const std::uint64_t end = std::min(n_ground, begin + kChunk);
    for (std::uint64_t p = begin; p < end;) {
      const double x = rng.uniform(0.0, ex);
      const double y = rng.uniform(0.0, ey);
      const double coin = rng.uniform01();
      if (!m.buildings.empty() && fp.covered(m, x, y)) continue;
      double z = terrain(m, x, y);
      if (coin < 0.3) z = z + rng.uniform(0.0, 20.0);
      xyz[3 * p + 0] = x;
      xyz[3 * p + 1] = y;
      xyz[3 * p + 2] = z;
      ++p;
    }
  });

  std::vector<std::uint64_t> start(m.buildings.size() + 1, n_ground);
  for (std::size_t b = 0; b < m.buildings.size(); ++b)
    start[b + 1] = start[b] + m.buildings[b].points;
  parallel_for(m.buildings.size(), T, [&](std::uint64_t b) {
    sample_building(m.buildings[b], seed, b, xyz + 3 * start[b]);
  });
  return 0;
}

// Uniform box [0,ex)x[0,ey)x[0,ez), bit-identical to the reference's
// SyntheticSpec::Kind::UniformBox (io.cpp:266-272): one mt19937_64 stream,
// x, y, z drawn in that order.
int cms_generate_uniform(uint64_t seed, uint64_t n, double ex, double ey,
                         double ez, double* xyz) {
  if (n == 0 || xyz == nullptr) return 2;
  Rng rng(seed);
  for (std::uint64_t i = 0; i < n; ++i) {
    xyz[3 * i + 0] = rng.uniform(0.0, ex);
    xyz[3 * i + 1] = rng.uniform(0.0, ey);
    xyz[3 * i + 2] = rng.uniform(0.0, ez);
  }
  return 0;
}

// The reference's SyntheticSpec kinds (io.cpp:252-335: UniformBox = 0,
// VoidEllipse = 1, GaussianClusters = 2), same RNG draws in the same order,
// same argument checks. Returns 0, or 2 (InvalidArgumentError) with the
// reference's message in msg.
int cms_generate_spec(int kind, uint64_t seed, uint64_t n, double ex, double ey, double ez,
                      double cx, double cy, double ax, double ay, uint64_t clusters,
                      double sigma, double* xyz, char* msg, int msglen) {
  auto fail = [&](const char* m) {
    if (msg && msglen > 0) {
      std::strncpy(msg, m, (size_t)msglen - 1);
      msg[msglen - 1] = 0;
    }
    return 2;
  };
  if (n == 0) return fail("synthetic point count must be positive");
  if (!(ex > 0.0) || !(ey > 0.0) || !(ez > 0.0)) return fail("synthetic extents must be positive");
  Rng rng(seed);
  uint64_t have = 0;
  auto push = [&](double x, double y, double z) {
    xyz[3 * have] = x, xyz[3 * have + 1] = y, xyz[3 * have + 2] = z;
    ++have;
  };
  if (kind == 0) {
    for (uint64_t i = 0; i < n; ++i) {
      const double x = rng.uniform(0.0, ex);
      const double y = rng.uniform(0.0, ey);
      push(x, y, rng.uniform(0.0, ez));
    }
    return 0;
  }
  if (kind == 1) {
    if (!(ax > 0.0) || !(ay > 0.0)) return fail("ellipse axes must be positive");
    if (cx - ax < 0.0 || cx + ax > ex || cy - ay < 0.0 || cy + ay > ey)
      return fail("void ellipse must lie inside the extents");
    uint64_t attempts = 0;
    const uint64_t max_attempts = n * 1000 + 1000;
    while (have < n) {
      if (++attempts > max_attempts) return fail("void region rejects nearly all samples; check the spec");
      const double x = rng.uniform(0.0, ex);
      const double y = rng.uniform(0.0, ey);
      const double u = (x - cx) / ax, v = (y - cy) / ay;
      if (u * u + v * v <= 1.0) continue;
      push(x, y, rng.uniform(0.0, ez));
    }
    return 0;
  }
  if (kind == 2) {
    if (clusters == 0 || !(sigma > 0.0)) return fail("need at least one cluster and sigma > 0");
    std::vector<double> c(3 * clusters);
    for (uint64_t i = 0; i < clusters; ++i) {
      c[3 * i] = rng.uniform(0.0, ex);
      c[3 * i + 1] = rng.uniform(0.0, ey);
      c[3 * i + 2] = rng.uniform(0.0, ez);
    }
    uint64_t attempts = 0;
    const uint64_t max_attempts = n * 1000 + 1000;
    while (have < n) {
      if (++attempts > max_attempts) return fail("cluster sampling rejects nearly all points; check sigma");
      const uint64_t k = rng.index(clusters);
      const double x = rng.gaussian(c[3 * k], sigma);
      const double y = rng.gaussian(c[3 * k + 1], sigma);
      const double z = rng.gaussian(c[3 * k + 2], sigma);
      if (x < 0.0 || x > ex || y < 0.0 || y > ey || z < 0.0 || z > ez) continue;
      push(x, y, z);
    }
    return 0;
  }
  return fail("unknown synthetic kind");
}

// TLS-like scan from (0, 0, scanner_z): n_az azimuths (2*pi*a/n_az) x n_el
// elevations (-60 deg + 120 deg * (e + 0.5) / n_el). Each ray returns its
// first hit among the ground plane z = 0 and n_boxes axis-aligned boxes
// (centres uniform in a 100 m disk, sides U[2,20] m, heights U[2,15] m,
// standing on z = 0, never containing the scanner), capped at max_range
// (rays with no hit, or a hit beyond it, return at max_range). Gaussian range
// noise sigma = noise_sigma from a per-ray splitmix64 stream. Output order is
// azimuth-major, elevation-minor. Returns 0 on success.
int cms_generate_tls(uint64_t seed, uint32_t n_az, uint32_t n_el,
                     uint32_t n_boxes, double scanner_z, double max_range,
                     double noise_sigma, uint32_t threads, double* xyz) {
  if (n_az == 0 || n_el == 0 || xyz == nullptr || !(max_range > 0.0)) return 2;
  struct Box {
    double x0, x1, y0, y1, z1;
    double a0, a1;  // azimuth interval [a0, a1] (radians, may wrap)
  };
  std::vector<Box> boxes;
  Rng rng(seed);
  while (boxes.size() < n_boxes) {
    const double rho = 100.0 * std::sqrt(rng.uniform01());
    const double ang = rng.uniform(0.0, kTwoPi);
    const double sx = rng.uniform(2.0, 20.0);
    const double sy = rng.uniform(2.0, 20.0);
    const double h = rng.uniform(2.0, 15.0);
    const double cx = rho * std::cos(ang), cy = rho * std::sin(ang);
    Box b{cx - sx / 2.0, cx + sx / 2.0, cy - sy / 2.0, cy + sy / 2.0, h, 0, 0};
    if (b.x0 - 1.0 <= 0.0 && b.x1 + 1.0 >= 0.0 && b.y0 - 1.0 <= 0.0 &&
        b.y1 + 1.0 >= 0.0)
      continue;  // scanner inside (or within 1 m of) the footprint
    // azimuth interval spanned by the four corners (the box does not
    // contain the origin, so it spans < pi)
    const double cs[4][2] = {{b.x0, b.y0}, {b.x0, b.y1}, {b.x1, b.y0}, {b.x1, b.y1}};
    const double ac = std::atan2(cy, cx);
    double lo = 0.0, hi = 0.0;
    for (auto& c : cs) {
      double d = std::atan2(c[1], c[0]) - ac;
      while (d > std::numbers::pi) d -= kTwoPi;
      while (d < -std::numbers::pi) d += kTwoPi;
      lo = std::min(lo, d);
      hi = std::max(hi, d);
    }
    b.a0 = ac + lo - 1e-9;
    b.a1 = ac + hi + 1e-9;
    boxes.push_back(b);
  }
  const unsigned T = worker_count(threads);
  // per-azimuth candidate box lists
  std::vector<std::vector<std::uint32_t>> cand(n_az);
  for (std::uint32_t a = 0; a < n_az; ++a) {
    const double az = kTwoPi * static_cast<double>(a) / static_cast<double>(n_az);
    for (std::uint32_t b = 0; b < boxes.size(); ++b) {
      double d = az - boxes[b].a0;
      while (d < 0.0) d += kTwoPi;
      while (d >= kTwoPi) d -= kTwoPi;
      if (d <= boxes[b].a1 - boxes[b].a0) cand[a].push_back(b);
    }
  }
  parallel_for(n_az, T, [&](std::uint64_t a) {
    const double az = kTwoPi * static_cast<double>(a) / static_cast<double>(n_az);
    const double ca = std::cos(az), sa = std::sin(az);
    for (std::uint32_t e = 0; e < n_el; ++e) {
      const double el = (-60.0 + 120.0 * (static_cast<double>(e) + 0.5) /
                                     static_cast<double>(n_el)) *
                        (std::numbers::pi / 180.0);
      const double dx = std::cos(el) * ca, dy = std::cos(el) * sa, dz = std::sin(el);
      double t = max_range;
      if (dz < 0.0) t = std::min(t, -scanner_z / dz);
      for (std::uint32_t b : cand[a]) {  // slab test, entry distance
        const Box& bx = boxes[b];
        double t0 = 0.0, t1 = t;
        const double o[3] = {0.0, 0.0, scanner_z};
        const double d[3] = {dx, dy, dz};
        const double lo[3] = {bx.x0, bx.y0, 0.0};
        const double hi[3] = {bx.x1, bx.y1, bx.z1};
        bool hit = true;
        for (int ax = 0; ax < 3 && hit; ++ax) {
          if (d[ax] == 0.0) {
            if (o[ax] < lo[ax] || o[ax] > hi[ax]) hit = false;
            continue;
          }
          double ta = (lo[ax] - o[ax]) / d[ax], tb = (hi[ax] - o[ax]) / d[ax];
          if (ta > tb) std::swap(ta, tb);
          t0 = std::max(t0, ta);
          t1 = std::min(t1, tb);
          if (t0 > t1) hit = false;
        }
        if (hit && t0 > 0.0) t = std::min(t, t0);
      }
      const std::uint64_t ray = a * static_cast<std::uint64_t>(n_el) + e;
      // Box-Muller from a counter-based stream (io.cpp:231-243 form)
      const std::uint64_t s1 = mix64(seed ^ mix64(2 * ray + 1));
      const std::uint64_t s2 = mix64(s1 ^ 0xd1b54a32d192ed03ull);
      const double u1 = static_cast<double>((s1 >> 11) + 1) * 0x1.0p-53;
      const double u2 = static_cast<double>(s2 >> 11) * 0x1.0p-53;
      const double g = std::sqrt(-2.0 * std::log(u1)) * std::cos(kTwoPi * u2);
      t = t + noise_sigma * g;
      xyz[3 * ray + 0] = t * dx;
      xyz[3 * ray + 1] = t * dy;
      xyz[3 * ray + 2] = scanner_z + t * dz;
    }
  });
  return 0;
}

// Query-centre indices, drawn with replacement: restates the reference CLI's
// CenterStream (tools/common.cpp:109-125): state = mix(seed ^ mix(tag));
// next: state = mix(state), index = state % cloud_size.
void cms_center_stream(uint64_t seed, uint64_t tag, uint64_t cloud_size,
                       uint64_t count, uint64_t* out) {
  std::uint64_t state = mix64(seed ^ mix64(tag));
  for (std::uint64_t i = 0; i < count; ++i) {
    state = mix64(state);
    out[i] = state % cloud_size;
  }
}

// The same stream as a resumable state (CenterStream, common.cpp:119-125).
uint64_t cms_center_stream_init(uint64_t seed, uint64_t tag) { return mix64(seed ^ mix64(tag)); }
void cms_center_stream_next(uint64_t* state, uint64_t cloud_size, uint64_t count, uint64_t* out) {
  std::uint64_t s = *state;
  for (std::uint64_t i = 0; i < count; ++i) {
    s = mix64(s);
    out[i] = s % cloud_size;
  }
  *state = s;
}

// Gather xyz of the given point indices (query centres drawn from a cloud).
void cms_gather_points(const double* xyz, const uint64_t* idx, uint64_t count,
                       double* out) {
  for (std::uint64_t i = 0; i < count; ++i) {
    std::memcpy(out + 3 * i, xyz + 3 * idx[i], 3 * sizeof(double));
  }
}

}  // extern "C"
