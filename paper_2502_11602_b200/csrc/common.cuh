// Shared device types and exact-arithmetic helpers for the sm_100a cheesemap
// engine. Every floating-point expression that decides a key or a membership
// uses explicit round-to-nearest intrinsics (no FMA contraction), and the
// whole library is also compiled with -fmad=false.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/cmgpu.h"

// Device-side invariant checks, compiled in only for the checked build
// (make checked -> libcmgpu_checked.so, CMGPU_LIB selects it): a failed check
// prints the condition and traps. The pool's GPUs have compute-sanitizer
// closed, so these plus CPU-oracle parity are the out-of-bounds evidence.
#ifdef CMGPU_CHECKED
#include <cstdio>
#define CM_DCHECK(cond)                                                            \
  do {                                                                             \
    if (!(cond)) {                                                                 \
      printf("CM_DCHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond);           \
      __trap();                                                                    \
    }                                                                              \
  } while (0)
#else
#define CM_DCHECK(cond) \
  do {                  \
  } while (0)
#endif

namespace cmg {

constexpr int kWarp = 32;
constexpr uint32_t kNone = 0xffffffffu;
constexpr uint64_t kEmptyKey = ~0ull;

// One stored point: fp64 xyz, the original handle and its voxel k (z index).
// 32 B, so a record is two aligned 16-byte loads and one L2 sector.
struct __align__(32) PointRec {
  double x, y, z;
  uint32_t id;
  uint32_t k;
};
static_assert(sizeof(PointRec) == 32, "record layout");

// GridParams (grid.hpp:47-81) as seen by kernels.
struct DevGrid {
  double ox, oy, oz;
  double sx, sy, sz;
  uint64_t nx, ny, nz;
  double bx0, by0, bz0, bx1, by1, bz1;
  int mode3d;
};

// Open-addressing slot: voxel key -> [a, b) point span, or column -> index.
struct __align__(16) HashSlot {
  uint64_t key;
  uint32_t a, b;
};

__host__ __device__ inline uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

// grid.cpp:29-37: idx = floor((coord - origin) / cell); <0 -> 0; min(idx, n-1)
__device__ __forceinline__ uint64_t axis_index(double coord, double origin, double cell,
                                               uint64_t n) {
  const double idx = floor(__ddiv_rn(__dsub_rn(coord, origin), cell));
  if (idx < 0.0) return 0;
  const uint64_t u = (uint64_t)idx;
  return u < n - 1 ? u : n - 1;
}

struct Range {
  uint64_t i0, i1, j0, j1, k0, k1;
};

// std::max / std::min exactly (NaN and signed-zero behaviour included).
__device__ __forceinline__ double std_max(double a, double b) { return (a < b) ? b : a; }
__device__ __forceinline__ double std_min(double a, double b) { return (b < a) ? b : a; }

// The query box of both kernels: c +- r per axis (geometry.hpp:77-80,
// cmd_bench.cpp:107-111), then clamped_range (grid.cpp:90-114) including the
// intersects() test against the bounds (geometry.hpp:53-56).
// Kernel kinds: 0 SphereKernel{c, r}, 1 BoxKernel{c - r, c + r}, 2 CylinderKernel
// {c.x, c.y, r} with an unbounded z range (geometry.hpp:97-113; its
// infinite box is clamped to the grid by clamped_range).
__device__ __forceinline__ void kernel_zbox(int kind, double cz, double r, double* lz, double* hz) {
  if (kind == 2) {
    *lz = __longlong_as_double(0xfff0000000000000ll);  // -inf
    *hz = __longlong_as_double(0x7ff0000000000000ll);  // +inf
  } else {
    *lz = __dsub_rn(cz, r);
    *hz = __dadd_rn(cz, r);
  }
}

// The kernel's box(): c +- r (sphere, cube, and the x / y extent of the
// cylinder), or, for queries given as explicit kernels (cm_kernel_search:
// BoxKernel's Aabb, CylinderKernel's z range), the caller's box
// {min xyz, max xyz}, which IS the reference's box() (geometry.hpp:87-113).
__device__ __forceinline__ void kernel_box(int kind, double cx, double cy, double cz, double r,
                                           const double* box, double* lx, double* ly, double* lz,
                                           double* hx, double* hy, double* hz) {
  if (box) {
    *lx = box[0], *ly = box[1], *lz = box[2];
    *hx = box[3], *hy = box[4], *hz = box[5];
    return;
  }
  *lx = __dsub_rn(cx, r), *hx = __dadd_rn(cx, r);
  *ly = __dsub_rn(cy, r), *hy = __dadd_rn(cy, r);
  kernel_zbox(kind, cz, r, lz, hz);
}

__device__ __forceinline__ bool clamped_range(const DevGrid& g, double cx, double cy, double cz,
                                              double r, Range* out, int kind = 0,
                                              const double* box = nullptr) {
  double lx, ly, lz, hx, hy, hz;
  kernel_box(kind, cx, cy, cz, r, box, &lx, &ly, &lz, &hx, &hy, &hz);
  if (!(lx <= g.bx1 && hx >= g.bx0 && ly <= g.by1 && hy >= g.by0 && lz <= g.bz1 &&
        hz >= g.bz0))
    return false;
  out->i0 = axis_index(std_max(lx, g.bx0), g.ox, g.sx, g.nx);
  out->i1 = axis_index(std_min(hx, g.bx1), g.ox, g.sx, g.nx);
  out->j0 = axis_index(std_max(ly, g.by0), g.oy, g.sy, g.ny);
  out->j1 = axis_index(std_min(hy, g.by1), g.oy, g.sy, g.ny);
  if (g.mode3d) {
    out->k0 = axis_index(std_max(lz, g.bz0), g.oz, g.sz, g.nz);
    out->k1 = axis_index(std_min(hz, g.bz1), g.oz, g.sz, g.nz);
  } else {
    out->k0 = out->k1 = 0;
  }
  return true;
}

// clamped_range computed by one warp for one (warp-uniform) query: lanes
// 0..5 each do one of the six IEEE divisions, then broadcast. Same
// arithmetic as clamped_range.
__device__ __forceinline__ bool clamped_range_warp(const DevGrid& g, double cx, double cy,
                                                   double cz, double r, int lane, Range* out,
                                                   int kind = 0, const double* box = nullptr) {
  double lx, ly, lz, hx, hy, hz;
  kernel_box(kind, cx, cy, cz, r, box, &lx, &ly, &lz, &hx, &hy, &hz);
  if (!(lx <= g.bx1 && hx >= g.bx0 && ly <= g.by1 && hy >= g.by0 && lz <= g.bz1 &&
        hz >= g.bz0))
    return false;
  uint64_t v = 0;
  if (lane < 6) {
    const int a = lane >> 1;
    const bool hi = lane & 1;
    const double c = a == 0 ? (hi ? std_min(hx, g.bx1) : std_max(lx, g.bx0))
                   : a == 1 ? (hi ? std_min(hy, g.by1) : std_max(ly, g.by0))
                            : (hi ? std_min(hz, g.bz1) : std_max(lz, g.bz0));
    const double o = a == 0 ? g.ox : a == 1 ? g.oy : g.oz;
    const double s = a == 0 ? g.sx : a == 1 ? g.sy : g.sz;
    const uint64_t n = a == 0 ? g.nx : a == 1 ? g.ny : g.nz;
    v = (a == 2 && !g.mode3d) ? 0 : axis_index(c, o, s, n);
  }
  out->i0 = __shfl_sync(0xffffffffu, v, 0);
  out->i1 = __shfl_sync(0xffffffffu, v, 1);
  out->j0 = __shfl_sync(0xffffffffu, v, 2);
  out->j1 = __shfl_sync(0xffffffffu, v, 3);
  out->k0 = __shfl_sync(0xffffffffu, v, 4);
  out->k1 = __shfl_sync(0xffffffffu, v, 5);
  return true;
}

// squared_distance (geometry.hpp:26-31): ((dx*dx + dy*dy) + dz*dz), dx = p - c
__device__ __forceinline__ double sqdist(double px, double py, double pz, double cx, double cy,
                                         double cz) {
  const double dx = __dsub_rn(px, cx);
  const double dy = __dsub_rn(py, cy);
  const double dz = __dsub_rn(pz, cz);
  return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
}

// Sphere (geometry.hpp:82-84) or closed cube (geometry.hpp:48-51).
struct Predicate {
  double cx, cy, cz;
  double rr;                          // r*r (sphere)
  double lx, ly, lz, hx, hy, hz;      // c -+ r (cube)
  int cube;

  __device__ __forceinline__ void init(double x, double y, double z, double r, int kind,
                                       const double* box = nullptr) {
    cx = x, cy = y, cz = z;
    rr = __dmul_rn(r, r);
    kernel_box(kind, x, y, z, r, box, &lx, &ly, &lz, &hx, &hy, &hz);
    cube = kind;
  }
  __device__ __forceinline__ bool operator()(double px, double py, double pz) const {
    if (cube)
      return px >= lx && px <= hx && py >= ly && py <= hy && pz >= lz && pz <= hz;
    return sqdist(px, py, pz, cx, cy, cz) <= rr;
  }
};

__device__ __forceinline__ PointRec load_rec(const PointRec* __restrict__ p) {
  const double2 a = __ldg(reinterpret_cast<const double2*>(p));
  const double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
  PointRec r;
  r.x = a.x;
  r.y = a.y;
  r.z = b.x;
  const uint2 t = *reinterpret_cast<const uint2*>(&b.y);
  r.id = t.x;
  r.k = t.y;
  return r;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ---------------------------------------------------------------- tables --

// Flavour-specific span lookup: the points of column (i, j) with voxel z
// index in [k0, k1] are ONE contiguous run of the cell-sorted records,
// because global_index is k-fastest (grid.hpp:65-67).
struct FRec;
struct Tables {
  DevGrid g;
  const PointRec* rec;
  const FRec* frec;       // float records (filter.cuh), same order as rec
  const uint32_t* ids;    // rec[].id, 4 B per record
  uint64_t n;
  int flavor;
  // dense: offsets over all V voxels (+1)
  const uint32_t* dense_off;
  // sparse: voxel hash key -> [begin, end)
  const HashSlot* vhash;
  uint64_t vmask;
  // mixed: column table (dense footprint array or hash) -> column c;
  // col_vbeg[c]..col_vbeg[c+1] unique voxels of column c; uk_k / ustart per
  // unique voxel.
  const uint32_t* col_dense;
  const HashSlot* chash;
  uint64_t cmask;
  const uint32_t* col_vbeg;
  const uint32_t* uk_k;
  const uint32_t* ustart;
};

__device__ __forceinline__ uint64_t hash_slot(uint64_t key, uint64_t mask) {
  return mix64(key) & mask;
}

__device__ __forceinline__ const HashSlot* hash_find(const HashSlot* t, uint64_t mask,
                                                     uint64_t key) {
  uint64_t s = hash_slot(key, mask);
  for (;;) {
    const HashSlot* e = t + s;
    const uint64_t k = __ldg(&e->key);
    if (k == key) return e;
    if (k == kEmptyKey) return nullptr;
    s = (s + 1) & mask;
  }
}

template <int FLAVOR>
__device__ __forceinline__ void column_span(const Tables& t, uint64_t i, uint64_t j, uint64_t k0,
                                            uint64_t k1, uint32_t* b, uint32_t* e) {
  const uint64_t nz = t.g.nz;
  if constexpr (FLAVOR == CM_DENSE) {
    const uint64_t g0 = (i * t.g.ny + j) * nz + k0;
    *b = __ldg(t.dense_off + g0);
    *e = __ldg(t.dense_off + g0 + (k1 - k0) + 1);
  } else if constexpr (FLAVOR == CM_SPARSE) {
    const uint64_t base = (i * t.g.ny + j) * nz;
    *b = *e = 0;
    uint64_t k = k0;
    const HashSlot* lo = nullptr;
    for (; k <= k1; ++k) {
      lo = hash_find(t.vhash, t.vmask, base + k);
      if (lo) break;
    }
    if (!lo) return;
    const HashSlot* hi = lo;
    for (uint64_t kk = k1; kk > k; --kk) {
      const HashSlot* h = hash_find(t.vhash, t.vmask, base + kk);
      if (h) {
        hi = h;
        break;
      }
    }
    *b = lo->a;
    *e = __ldg(&hi->b);
  } else {
    const uint64_t col = i * t.g.ny + j;
    uint32_t c;
    if (t.col_dense) {
      c = __ldg(t.col_dense + col);
    } else {
      const HashSlot* h = hash_find(t.chash, t.cmask, col);
      c = h ? __ldg(&h->a) : kNone;
    }
    *b = *e = 0;
    if (c == kNone) return;
    uint32_t v0 = __ldg(t.col_vbeg + c), v1 = __ldg(t.col_vbeg + c + 1);
    // first voxel with k >= k0, first voxel with k > k1 (k ascending)
    uint32_t lo = v0, hi = v1;
    while (lo < hi) {
      const uint32_t m = (lo + hi) >> 1;
      if (__ldg(t.uk_k + m) < k0) lo = m + 1; else hi = m;
    }
    uint32_t lo2 = lo, hi2 = v1;
    while (lo2 < hi2) {
      const uint32_t m = (lo2 + hi2) >> 1;
      if (__ldg(t.uk_k + m) <= k1) lo2 = m + 1; else hi2 = m;
    }
    if (lo2 == lo) return;
    *b = __ldg(t.ustart + lo);
    *e = __ldg(t.ustart + lo2);
  }
}

}  // namespace cmg

// ----------------------------------------------------------- host helpers --

namespace cmg {
void set_error(const std::string& msg);
// Counts every kernel this library launches (cm_launch_count).
void note_launch();
}

#define CM_CUDA_TRY(expr)                                                         \
  do {                                                                            \
    cudaError_t _e = (expr);                                                      \
    if (_e != cudaSuccess) {                                                      \
      ::cmg::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));       \
      return CM_CUDA;                                                             \
    }                                                                             \
  } while (0)
