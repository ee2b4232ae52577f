// Filtered exact predicates: an fp32 estimate that decides every candidate
// whose outcome it can prove, and the reference's exact fp64 arithmetic
// (common.cuh sqdist / closed box, geometry.hpp:26-31,48-51,82-84) for the
// rest. Results are bit-identical to the fp64 predicate; only the cost
// changes (DESIGN.md §3 "Filtered predicates").
//
// Float records (FRec, 16 B, cell order like PointRec): x and y relative to
// the record's column corner C = o + i * s (fp64, then rounded to fp32), z
// relative to the grid origin oz, and the voxel k. A lane answering centre c
// forms, per staged chunk of column (i, j), B = C - c in fp64 once, and per
// record d_f = fl32(A_f + B_f). With u = 2^-24 and every |A|, |B| bounded,
//   |d_f,a - d_a| <= 2^-22.9 (|A_a| + |B_a|)   per axis,
// so ||d_f - d|| <= eps = 2^-22 * sum_a (Amax_a + Bmax_a) (eps_of below).
// The fp32 d2_f = fma(dz, dz, fma(dy, dy, dx * dx)) has relative error
// <= 3u < 2^-22. The thresholds then prove (filter_init):
//   d2_f <= tin   =>  the fp64 predicate holds (||d|| <= r (1 - 2^-48), and
//                     the fp64 sqdist is within (1 + 2^-50) of ||d||^2, while
//                     fl(r * r) >= r^2 (1 - 2^-53));
//   d2_f >  tout  =>  it fails (||d|| > r (1 + 2^-48));
// anything between is decided by the exact fp64 predicate on the record's
// fp64 coordinates. The cube (closed box fl(c -+ r)) uses max_a |d_f,a|
// against r -+ (eps + 2^-52 (|c| + r)). NaN anywhere makes every comparison
// false on both paths. Radii outside [2^-400, 2^400] disable the filter.
#pragma once

#include "common.cuh"

// Filtered predicates in the compact tile walk (and the float records the
// build writes for them): measured slower at r = 1 (collect 9.9 -> 11.3 ms),
// so compiled in only on request (-DCM_FILTER=1).
#ifndef CM_FILTER
#define CM_FILTER 0
#endif

namespace cmg {

struct __align__(16) FRec {
  float x, y, z;
  uint32_t k;
};
static_assert(sizeof(FRec) == 16, "float record layout");

// Column corner o + i * s, computed identically at build and query time.
__host__ __device__ __forceinline__ double col_corner(double o, uint64_t i, double s) {
#ifdef __CUDA_ARCH__
  return __dadd_rn(o, __dmul_rn((double)i, s));
#else
  return o + (double)i * s;
#endif
}

// Per-lane filter state for one tile (hull columns I0.., J0.., nI x nJ).
struct Filter {
  float az;          // fl32(oz - cz)
  float tin, tout;   // sphere: bounds on d2_f; cube: bounds on max |d_f|
  double cx, cy;     // the centre (per-chunk column offsets)
};

// eps for a centre whose candidate columns span [I0, I0 + nI) x [J0, J0 + nJ).
__device__ __forceinline__ double eps_of(const DevGrid& g, double cx, double cy, double cz,
                                         uint64_t I0, uint64_t nI, uint64_t J0, uint64_t nJ) {
  const double bx = fabs(col_corner(g.ox, I0, g.sx) - cx) + (double)(nI + 1) * g.sx;
  const double by = fabs(col_corner(g.oy, J0, g.sy) - cy) + (double)(nJ + 1) * g.sy;
  const double bz = fabs(g.oz - cz);
  const double zext = g.bz1 - g.bz0;
  // |A_x| <= s_x (1 + tiny), |A_z| <= zext; 1.01 and the 2^-22 factor are
  // generous against the 2^-22.9 bound and this function's own rounding
  return 0x1p-22 * 1.01 * (1.01 * g.sx + bx + 1.01 * g.sy + by + zext + bz);
}

// CUBE: 0 sphere, 1 closed cube; anything else (cylinder, explicit boxes)
// never reaches the filter.
template <int CUBE>
__device__ __forceinline__ void filter_init(Filter& F, const DevGrid& g, double cx, double cy,
                                            double cz, double r, double eps) {
  F.cx = cx, F.cy = cy;
  F.az = __double2float_rn(__dsub_rn(g.oz, cz));
  const bool usable = r >= 0x1p-400 && r <= 0x1p400 && eps < 0x1p400;
  if (CUBE == 1) {
    const double cm = fmax(fabs(cx), fmax(fabs(cy), fabs(cz)));
    const double slack = 0x1p-52 * (cm + r) + eps;
    const double lo = r - slack, hi = r + slack;
    F.tin = (usable && lo > 0.0) ? __double2float_rd(lo * (1.0 - 0x1p-40)) : -1.0f;
    F.tout = usable ? __double2float_ru(hi * (1.0 + 0x1p-40)) : __int_as_float(0x7f800000);
  } else {
    const double rlo = r * (1.0 - 0x1p-48) - eps;
    const double rhi = r * (1.0 + 0x1p-48) + eps;
    F.tin = (usable && rlo > 0.0) ? __double2float_rd((1.0 - 0x1p-22) * rlo * rlo) : -1.0f;
    F.tout = usable ? __double2float_ru((1.0 + 0x1p-22) * rhi * rhi) : __int_as_float(0x7f800000);
  }
}

// The filter's value for a record at float offsets (dx, dy, dz) from the centre.
template <int CUBE>
__device__ __forceinline__ float filter_value(float dx, float dy, float dz) {
  if (CUBE == 1) return fmaxf(fabsf(dx), fmaxf(fabsf(dy), fabsf(dz)));
  return __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
}

}  // namespace cmg
