// Exact batched kNN on sm_100a, ordered by (fp64 squared distance, handle).
// Replaces knn_search (search.cpp:87-146).
//
// The reference grows a ball by a density estimate (grow_radius,
// search.cpp:58-74) and stops when k candidates lie within the visited
// radius. Here a warp walks Chebyshev voxel shells around the centre's voxel
// (shell L = voxels at max(|di|,|dj|,|dk|) == L; ring columns contribute
// their whole z range, inner columns only k0 +- L) and stops once the k-th
// best squared distance is strictly below the squared distance from the
// centre to every unvisited voxel (less a rounding margin). Both searches are
// exact; this one also settles ties by handle, which the reference's
// insertion-ordered CandidateList (search.cpp:16-28) does not.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

#include "index.cuh"
#include "sort_scan.cuh"
#include "tile_walk.cuh"

namespace cmg {

namespace {

constexpr int kKThreads = 128;
constexpr int kKWarps = kKThreads / 32;
constexpr int kKMax = 256;
#ifndef CM_KNN_TILE_MAX
#define CM_KNN_TILE_MAX 8
#endif
constexpr uint32_t kKnnTileMax = CM_KNN_TILE_MAX;  // kNN query tiles for k <= this

__device__ __forceinline__ int64_t imax64(int64_t a, int64_t b) { return a < b ? b : a; }
__device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return b < a ? b : a; }

__device__ __forceinline__ bool pair_less(double a, uint32_t ia, double b, uint32_t ib) {
  return a < b || (a == b && ia < ib);
}

// 32-wide bitonic sort of (d2, handle) pairs, one per lane, ascending by lane.
__device__ __forceinline__ void warp_sort_pairs32(double& d, uint32_t& id, int lane) {
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const double od = __shfl_xor_sync(0xffffffffu, d, j);
      const uint32_t oi = __shfl_xor_sync(0xffffffffu, id, j);
      const bool up = (lane & k) == 0 || k == 32;
      const bool lower = (lane & j) == 0;
      const bool o_less = pair_less(od, oi, d, id);
      const bool take_o = (lower == up) ? o_less : !o_less;
      d = take_o ? od : d;
      id = take_o ? oi : id;
    }
  }
}

template <int FLAVOR>
__device__ __forceinline__ void shell_column_spans(const Tables& t, int64_t i, int64_t j,
                                                   bool ring, int64_t kc, int64_t L,
                                                   uint64_t kmax, uint32_t* b1, uint32_t* e1,
                                                   uint32_t* b2, uint32_t* e2) {
  *b1 = *e1 = *b2 = *e2 = 0;
  if (ring) {
    const int64_t k0 = imax64(0, kc - L);
    const int64_t k1 = imin64((int64_t)kmax, kc + L);
    column_span<FLAVOR>(t, (uint64_t)i, (uint64_t)j, (uint64_t)k0, (uint64_t)k1, b1, e1);
  } else {
    if (kc - L >= 0)
      column_span<FLAVOR>(t, (uint64_t)i, (uint64_t)j, (uint64_t)(kc - L), (uint64_t)(kc - L), b1, e1);
    if (kc + L <= (int64_t)kmax)
      column_span<FLAVOR>(t, (uint64_t)i, (uint64_t)j, (uint64_t)(kc + L), (uint64_t)(kc + L), b2, e2);
  }
}

// Radius-box walk in the per-thread kernel (CMGPU_KNN_R0MULT > 0 at run
// time): exact, measured slower than the shells on config 3 (k = 8: 10.4 ->
// 13.4 ms at 1.3 x the expected k-th distance); compiled in only on request.
#ifndef CM_KNN_TBATCH
#define CM_KNN_TBATCH 2  // records in flight per thread (per-thread kNN walk)
#endif
#ifndef CM_KNN_TMINB
#define CM_KNN_TMINB 10  // blocks per SM the per-thread kernel is compiled for (k <= 16)
#endif
#ifndef CM_KNN_TMINB8
#define CM_KNN_TMINB8 12  // the same for k <= 8 (12 KB of heaps per block: config 3 k = 8 5.54 -> 5.40 ms)
#endif
#ifndef CM_KNN_BOX
#define CM_KNN_BOX 0
#endif
#ifndef CM_KNN_PRUNE
#define CM_KNN_PRUNE 2  // per-thread kernel: 0 whole block, 1 pruned columns, 2 pruned + nearest first
#endif
#ifndef CM_KNN_BALL
#define CM_KNN_BALL 0  // measured slower on config 3 (k = 64: 39.3 -> 47.8 ms): opt-in
#endif
constexpr bool kBallWarp = CM_KNN_BALL;  // ball completion in the shell walk

// GLIST = false: the sorted (d2, handle) list of one query lives in shared
// memory (k <= kKMax). GLIST = true (any k): it lives in the outputs
// themselves (idx_out row, and d2_out row or a chunk-local d2 scratch).
template <int FLAVOR, bool GLIST>
__global__ void __launch_bounds__(kKThreads) knn_warp_kernel(const Tables t,
                                                             const double* __restrict__ q,
                                                             uint64_t s_begin, uint64_t s_end,
                                                             uint32_t k,
                                                             const uint32_t* __restrict__ perm,
                                                             uint32_t* __restrict__ idx_out,
                                                             double* __restrict__ d2_out,
                                                             double* __restrict__ d2_scratch,
                                                             const uint32_t* __restrict__ n_dev) {
  if (n_dev) s_end = s_end < (uint64_t)*n_dev ? s_end : (uint64_t)*n_dev;  // a device-built redo list
  // the sorted list and, for batch merges, its second buffer
  __shared__ double sd[GLIST ? 1 : kKWarps][2][GLIST ? 1 : kKMax];
  __shared__ uint32_t sid[GLIST ? 1 : kKWarps][2][GLIST ? 1 : kKMax];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  double* ld = sd[GLIST ? 0 : wib][0];
  uint32_t* lid = sid[GLIST ? 0 : wib][0];
  double* ld2 = sd[GLIST ? 0 : wib][1];
  uint32_t* lid2 = sid[GLIST ? 0 : wib][1];
  const uint64_t W = (uint64_t)gridDim.x * kKWarps;
  const DevGrid& g = t.g;
  const uint32_t lt = lanemask_lt();
  const int64_t nx = (int64_t)g.nx, ny = (int64_t)g.ny, nzm = (int64_t)g.nz - 1;

  for (uint64_t s = s_begin + (uint64_t)blockIdx.x * kKWarps + wib; s < s_end; s += W) {
    const uint32_t qi = perm ? __ldg(perm + s) : (uint32_t)s;
    if (GLIST) {
      lid = idx_out + (uint64_t)qi * k;
      ld = d2_out ? d2_out + (uint64_t)qi * k : d2_scratch + (s - s_begin) * k;
    }
    const double cx = __ldg(q + 3 * (uint64_t)qi);
    const double cy = __ldg(q + 3 * (uint64_t)qi + 1);
    const double cz = __ldg(q + 3 * (uint64_t)qi + 2);
    const int64_t ic = (int64_t)axis_index(cx, g.ox, g.sx, g.nx);
    const int64_t jc = (int64_t)axis_index(cy, g.oy, g.sy, g.ny);
    const int64_t kc = g.mode3d ? (int64_t)axis_index(cz, g.oz, g.sz, g.nz) : 0;
    // rounding margin for the unvisited-distance bound (coordinates ulps)
    const double eps = 1e-12 * (fabs(cx) + fabs(cy) + fabs(cz) + fabs(g.ox) + fabs(g.oy) +
                                fabs(g.oz) + g.sx + g.sy + g.sz);
    uint32_t cnt = 0;
    // The first step visits the whole 3 x 3 x 3 block (shells 0 and 1 at
    // once: the shell-0 stop test almost never holds for k >= 8 at
    // cell-sized voxels, so testing it only cost a round of span lookups and
    // a batch merge); later steps add one Chebyshev shell each.
    // Columns [0, ncol) of a visit set, 32 per step: spans(c, ...) gives
    // column c's (at most two) record spans.
    auto walk_cols = [&](uint32_t ncol, auto spans) {
      for (uint32_t cb = 0; cb < ncol; cb += 32) {
        const uint32_t c = cb + lane;
        uint32_t b1 = 0, e1 = 0, b2 = 0, e2 = 0;
        if (c < ncol) spans(c, &b1, &e1, &b2, &e2);
        const uint32_t l1 = e1 - b1;
        const uint32_t len = l1 + (e2 - b2);
        const uint32_t incl = warp_incl_scan(len);
        const uint32_t excl = incl - len;
        const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
        for (uint32_t t0 = 0; t0 < total; t0 += 32) {
          const uint32_t tt = t0 + lane;
          int Lq = 0;
#pragma unroll
          for (int sft = 16; sft > 0; sft >>= 1) {
            const uint32_t v = __shfl_sync(0xffffffffu, incl, Lq + sft - 1);
            if (v <= tt) Lq += sft;
          }
          const uint32_t xL = __shfl_sync(0xffffffffu, excl, Lq);
          const uint32_t b1L = __shfl_sync(0xffffffffu, b1, Lq);
          const uint32_t l1L = __shfl_sync(0xffffffffu, l1, Lq);
          const uint32_t b2L = __shfl_sync(0xffffffffu, b2, Lq);
          double d2 = 0.0;
          uint32_t id = 0;
          bool acc = false;
          if (tt < total) {
            const uint32_t o = tt - xL;
            const uint32_t pos = o < l1L ? b1L + o : b2L + (o - l1L);
            const PointRec pr = load_rec(t.rec + pos);
            d2 = sqdist(pr.x, pr.y, pr.z, cx, cy, cz);
            id = pr.id;
            acc = cnt < k || pair_less(d2, id, ld[k - 1], lid[k - 1]);
          }
          uint32_t m = __ballot_sync(0xffffffffu, acc);
          const uint32_t nacc = __popc(m);
          if (!GLIST && nacc > 0) {
            // batch merge: sort the accepted candidates, then place every
            // list and batch entry at (own index + its rank in the other
            // sequence) in the second buffer, keeping the k smallest
            double bd = acc ? d2 : __longlong_as_double(0x7ff0000000000000ll);
            uint32_t bi = acc ? id : 0xffffffffu;
            warp_sort_pairs32(bd, bi, lane);
            const uint32_t ncnt = min(k, cnt + nacc);
            CM_DCHECK(ncnt <= (uint32_t)kKMax);
            for (uint32_t base = 0; base < cnt; base += 32) {
              const uint32_t x = base + lane;
              const bool valid = x < cnt;
              const double xd = valid ? ld[x] : 0.0;
              const uint32_t xi = valid ? lid[x] : 0u;
              uint32_t r = 0;
#pragma unroll
              for (int sft = 16; sft > 0; sft >>= 1) {
                const double od = __shfl_sync(0xffffffffu, bd, r + sft - 1);
                const uint32_t oi = __shfl_sync(0xffffffffu, bi, r + sft - 1);
                if (pair_less(od, oi, xd, xi)) r += sft;
              }
              const double od = __shfl_sync(0xffffffffu, bd, 31);
              const uint32_t oi = __shfl_sync(0xffffffffu, bi, 31);
              if (r == 31 && pair_less(od, oi, xd, xi)) r = 32;
              if (valid && x + r < ncnt) {
                ld2[x + r] = xd;
                lid2[x + r] = xi;
              }
            }
            if ((uint32_t)lane < nacc) {
              uint32_t lo = 0, hi = cnt;
              while (lo < hi) {
                const uint32_t mid = (lo + hi) >> 1;
                if (pair_less(ld[mid], lid[mid], bd, bi)) lo = mid + 1; else hi = mid;
              }
              if (lane + lo < ncnt) {
                ld2[lane + lo] = bd;
                lid2[lane + lo] = bi;
              }
            }
            __syncwarp();
            double* td = ld;
            ld = ld2;
            ld2 = td;
            uint32_t* ti = lid;
            lid = lid2;
            lid2 = ti;
            cnt = ncnt;
            m = 0;
          }
          while (m) {
            const int src = __ffs(m) - 1;
            m &= m - 1;
            const double d = __shfl_sync(0xffffffffu, d2, src);
            const uint32_t di = __shfl_sync(0xffffffffu, id, src);
            if (cnt == k && !pair_less(d, di, ld[k - 1], lid[k - 1])) continue;
            // insertion position = #entries less than (d, di)
            uint32_t pos = 0;
            for (uint32_t base = 0; base < cnt; base += 32) {
              const uint32_t x = base + lane;
              const bool less = x < cnt && pair_less(ld[x], lid[x], d, di);
              pos += __popc(__ballot_sync(0xffffffffu, less));
            }
            const uint32_t ncnt = cnt < k ? cnt + 1 : k;
            // shift [pos, ncnt-1) -> [pos+1, ncnt), 32 slots at a time from
            // the top (each chunk reads below itself before it is written)
            for (int64_t top = (int64_t)ncnt - 1; top > (int64_t)pos; top -= 32) {
              const int64_t x = top - lane;
              double vd = 0.0;
              uint32_t vi = 0;
              const bool mv = x > (int64_t)pos;
              if (mv) {
                vd = ld[x - 1];
                vi = lid[x - 1];
              }
              __syncwarp();
              if (mv) {
                ld[x] = vd;
                lid[x] = vi;
              }
              __syncwarp();
            }
            if (lane == 0) {
              ld[pos] = d;
              lid[pos] = di;
            }
            __syncwarp();
            cnt = ncnt;
          }
        }
      }
    };
    for (int64_t L = 1;; ++L) {
      const int64_t i0 = imax64(0, ic - L), i1 = imin64(nx - 1, ic + L);
      const int64_t j0 = imax64(0, jc - L), j1 = imin64(ny - 1, jc + L);
      const uint32_t nj = (uint32_t)(j1 - j0 + 1);
      const uint32_t ncol = (uint32_t)(i1 - i0 + 1) * nj;
      walk_cols(ncol, [&](uint32_t c, uint32_t* b1, uint32_t* e1, uint32_t* b2, uint32_t* e2) {
        const int64_t i = i0 + (int64_t)(c / nj), j = j0 + (int64_t)(c % nj);
        const bool ring = L == 1 || (i == ic - L) || (i == ic + L) || (j == jc - L) || (j == jc + L);
        shell_column_spans<FLAVOR>(t, i, j, ring, kc, L, (uint64_t)nzm, b1, e1, b2, e2);
      });
      // distance from c to the nearest unvisited voxel face
      const bool all = i0 == 0 && i1 == nx - 1 && j0 == 0 && j1 == ny - 1 &&
                       imax64(0, kc - L) == 0 && imin64(nzm, kc + L) == nzm;
      if (all) break;
      if (cnt == k) {
        double dmin = 1e300;
        if (i0 > 0) dmin = fmin(dmin, cx - (g.ox + (double)i0 * g.sx));
        if (i1 < nx - 1) dmin = fmin(dmin, (g.ox + (double)(i1 + 1) * g.sx) - cx);
        if (j0 > 0) dmin = fmin(dmin, cy - (g.oy + (double)j0 * g.sy));
        if (j1 < ny - 1) dmin = fmin(dmin, (g.oy + (double)(j1 + 1) * g.sy) - cy);
        if (g.mode3d) {
          if (kc - L > 0) dmin = fmin(dmin, cz - (g.oz + (double)(kc - L) * g.sz));
          if (kc + L < nzm) dmin = fmin(dmin, (g.oz + (double)(kc + L + 1) * g.sz) - cz);
        }
        const double dm = dmin - eps;
        if (dm > 0.0 && ld[k - 1] < dm * dm) break;
        // Ball completion instead of the next whole shell: every voxel of
        // clamped_range(c +- R) outside the visited block, R = the current
        // k-th distance rounded up (a point that beats the final k-th has
        // fp64 d² <= kd, true distance <= sqrt(kd)(1 + 2^-51) <= R, and
        // axis_index is monotone): exact, and the walk ends here.
        if (kBallWarp) {
          const double R = sqrt(ld[k - 1]) * (1.0 + 1e-12) + eps;
          Range B;
          if (clamped_range(g, cx, cy, cz, R, &B, 0)) {
            const uint32_t bnj = (uint32_t)(B.j1 - B.j0 + 1);
            const uint32_t bnc = (uint32_t)(B.i1 - B.i0 + 1) * bnj;
            walk_cols(bnc, [&](uint32_t c, uint32_t* b1, uint32_t* e1, uint32_t* b2, uint32_t* e2) {
              const int64_t i = (int64_t)B.i0 + (int64_t)(c / bnj), j = (int64_t)B.j0 + (int64_t)(c % bnj);
              const bool inblock = i >= ic - L && i <= ic + L && j >= jc - L && j <= jc + L;
              int64_t lo1 = (int64_t)B.k0, hi1 = (int64_t)B.k1, lo2 = 1, hi2 = 0;
              if (inblock) {  // only the parts below and above the block
                hi1 = imin64(hi1, kc - L - 1);
                lo2 = imax64((int64_t)B.k0, kc + L + 1);
                hi2 = (int64_t)B.k1;
              }
              if (lo1 <= hi1)
                column_span<FLAVOR>(t, (uint64_t)i, (uint64_t)j, (uint64_t)lo1, (uint64_t)hi1, b1, e1);
              if (lo2 <= hi2)
                column_span<FLAVOR>(t, (uint64_t)i, (uint64_t)j, (uint64_t)lo2, (uint64_t)hi2, b2, e2);
            });
          }
          break;
        }
      }
    }
    if (GLIST) {
      for (uint32_t x = cnt + lane; x < k; x += 32) {
        lid[x] = 0xffffffffu;
        ld[x] = __longlong_as_double(0x7ff0000000000000ll);
      }
    } else {
      for (uint32_t x = lane; x < k; x += 32) {
        idx_out[(uint64_t)qi * k + x] = x < cnt ? lid[x] : 0xffffffffu;
        if (d2_out)
          d2_out[(uint64_t)qi * k + x] = x < cnt ? ld[x] : __longlong_as_double(0x7ff0000000000000ll);
      }
    }
    __syncwarp();
  }
  (void)lt;
}

// One warp per centre with the sorted (d², handle) list in REGISTERS (k <= 32):
// lane l holds the l-th best entry, pads are (inf, 0xffffffff) — the output
// convention for missing neighbours. The walk is knn_warp_kernel's (lanes
// look up one column each, candidates flattened 32 per step); a step's
// accepted candidates enter the list one by one (rank by ballot, shift by
// shuffle: no shared memory) or, when there are many, sorted and merged
// through the bitonic half-cleaner (the 32 smallest of two sorted 32-lists
// are min(A[l], B[31 - l]), a bitonic sequence). Used for the centres the
// per-thread kernel's first pass cannot finish (sparse neighbourhoods: many
// span lookups, few candidates), and for 16 < k <= 32.
#ifndef CM_KNN_SORTMIN
#define CM_KNN_SORTMIN 12  // accepted candidates per step from which the batch is sorted and merged
#endif
#ifndef CM_KNN_REG_MINB
#define CM_KNN_REG_MINB 8  // 64 registers (an explicit 1 lets ptxas take far more: slower)
#endif
template <int FLAVOR>
__global__ void __launch_bounds__(kKThreads, CM_KNN_REG_MINB) knn_warp_reg_kernel(
    const Tables t, const double* __restrict__ q, uint64_t s_begin, uint64_t s_end, uint32_t k,
    const uint32_t* __restrict__ perm, uint32_t* __restrict__ idx_out, double* __restrict__ d2_out,
    const uint32_t* __restrict__ n_dev, int L0) {
  // L0: the first step visits the whole Chebyshev-L0 block (one span lookup
  // per column); the pass-2 centres are known to need more than the 3 x 3 x 3
  // block, so they start at L0 = 2: one round of lookups less
  if (n_dev) s_end = s_end < (uint64_t)*n_dev ? s_end : (uint64_t)*n_dev;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const uint64_t W = (uint64_t)gridDim.x * kKWarps;
  const DevGrid& g = t.g;
  const int64_t nx = (int64_t)g.nx, ny = (int64_t)g.ny, nzm = (int64_t)g.nz - 1;
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);
  for (uint64_t s = s_begin + (uint64_t)blockIdx.x * kKWarps + wib; s < s_end; s += W) {
    const uint32_t qi = perm ? __ldg(perm + s) : (uint32_t)s;
    const double cx = __ldg(q + 3 * (uint64_t)qi);
    const double cy = __ldg(q + 3 * (uint64_t)qi + 1);
    const double cz = __ldg(q + 3 * (uint64_t)qi + 2);
    const int64_t ic = (int64_t)axis_index(cx, g.ox, g.sx, g.nx);
    const int64_t jc = (int64_t)axis_index(cy, g.oy, g.sy, g.ny);
    const int64_t kc = g.mode3d ? (int64_t)axis_index(cz, g.oz, g.sz, g.nz) : 0;
    const double eps = 1e-12 * (fabs(cx) + fabs(cy) + fabs(cz) + fabs(g.ox) + fabs(g.oy) +
                                fabs(g.oz) + g.sx + g.sy + g.sz);
    double rd = kInf;  // this lane's list entry
    uint32_t ri = 0xffffffffu;
    double kd = kInf;  // entry k - 1 (warp-uniform)
    uint32_t kid = 0xffffffffu;
    auto walk_cols = [&](uint32_t ncol, auto spans) {
      for (uint32_t cb = 0; cb < ncol; cb += 32) {
        const uint32_t c = cb + lane;
        uint32_t b1 = 0, e1 = 0, b2 = 0, e2 = 0;
        if (c < ncol) spans(c, &b1, &e1, &b2, &e2);
        const uint32_t l1 = e1 - b1;
        const uint32_t len = l1 + (e2 - b2);
        const uint32_t incl = warp_incl_scan(len);
        const uint32_t excl = incl - len;
        const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
        for (uint32_t t0 = 0; t0 < total; t0 += 32) {
          const uint32_t tt = t0 + lane;
          int Lq = 0;
#pragma unroll
          for (int sft = 16; sft > 0; sft >>= 1) {
            const uint32_t v = __shfl_sync(0xffffffffu, incl, Lq + sft - 1);
            if (v <= tt) Lq += sft;
          }
          const uint32_t xL = __shfl_sync(0xffffffffu, excl, Lq);
          const uint32_t b1L = __shfl_sync(0xffffffffu, b1, Lq);
          const uint32_t l1L = __shfl_sync(0xffffffffu, l1, Lq);
          const uint32_t b2L = __shfl_sync(0xffffffffu, b2, Lq);
          double d2 = kInf;
          uint32_t id = 0xffffffffu;
          bool acc = false;
          if (tt < total) {
            const uint32_t o = tt - xL;
            const uint32_t pos = o < l1L ? b1L + o : b2L + (o - l1L);
            const PointRec pr = load_rec(t.rec + pos);
            d2 = sqdist(pr.x, pr.y, pr.z, cx, cy, cz);
            id = pr.id;
            acc = pair_less(d2, id, kd, kid);
          }
          uint32_t m = __ballot_sync(0xffffffffu, acc);
          if (!m) continue;
          if (__popc(m) >= CM_KNN_SORTMIN) {
            double bd = acc ? d2 : kInf;
            uint32_t bi = acc ? id : 0xffffffffu;
            warp_sort_pairs32(bd, bi, lane);
            const double od = __shfl_sync(0xffffffffu, bd, 31 - lane);
            const uint32_t oi = __shfl_sync(0xffffffffu, bi, 31 - lane);
            if (pair_less(od, oi, rd, ri)) rd = od, ri = oi;
#pragma unroll
            for (int j = 16; j > 0; j >>= 1) {
              const double pd = __shfl_xor_sync(0xffffffffu, rd, j);
              const uint32_t pi = __shfl_xor_sync(0xffffffffu, ri, j);
              const bool p_less = pair_less(pd, pi, rd, ri);
              const bool take = ((lane & j) == 0) ? p_less : !p_less;
              rd = take ? pd : rd;
              ri = take ? pi : ri;
            }
          } else {
            while (m) {
              const int src = __ffs(m) - 1;
              m &= m - 1;
              const double d = __shfl_sync(0xffffffffu, d2, src);
              const uint32_t di = __shfl_sync(0xffffffffu, id, src);
              // rank among the 32 entries: lanes holding smaller entries are a prefix
              const uint32_t pos = __popc(__ballot_sync(0xffffffffu, pair_less(rd, ri, d, di)));
              const double ud = __shfl_up_sync(0xffffffffu, rd, 1);
              const uint32_t ui = __shfl_up_sync(0xffffffffu, ri, 1);
              if ((uint32_t)lane > pos) rd = ud, ri = ui;
              if ((uint32_t)lane == pos) rd = d, ri = di;
            }
          }
          kd = __shfl_sync(0xffffffffu, rd, (int)k - 1);
          kid = __shfl_sync(0xffffffffu, ri, (int)k - 1);
        }
      }
    };
    for (int64_t L = L0;; ++L) {
      const int64_t i0 = imax64(0, ic - L), i1 = imin64(nx - 1, ic + L);
      const int64_t j0 = imax64(0, jc - L), j1 = imin64(ny - 1, jc + L);
      const uint32_t nj = (uint32_t)(j1 - j0 + 1);
      const uint32_t ncol = (uint32_t)(i1 - i0 + 1) * nj;
      walk_cols(ncol, [&](uint32_t c, uint32_t* b1, uint32_t* e1, uint32_t* b2, uint32_t* e2) {
        const int64_t i = i0 + (int64_t)(c / nj), j = j0 + (int64_t)(c % nj);
        const bool ring = L == L0 || (i == ic - L) || (i == ic + L) || (j == jc - L) || (j == jc + L);
        shell_column_spans<FLAVOR>(t, i, j, ring, kc, L, (uint64_t)nzm, b1, e1, b2, e2);
      });
      const bool all = i0 == 0 && i1 == nx - 1 && j0 == 0 && j1 == ny - 1 &&
                       imax64(0, kc - L) == 0 && imin64(nzm, kc + L) == nzm;
      if (all) break;
      if (kid != 0xffffffffu) {  // k entries known: the shell walk's stop test
        double dmin = 1e300;
        if (i0 > 0) dmin = fmin(dmin, cx - (g.ox + (double)i0 * g.sx));
        if (i1 < nx - 1) dmin = fmin(dmin, (g.ox + (double)(i1 + 1) * g.sx) - cx);
        if (j0 > 0) dmin = fmin(dmin, cy - (g.oy + (double)j0 * g.sy));
        if (j1 < ny - 1) dmin = fmin(dmin, (g.oy + (double)(j1 + 1) * g.sy) - cy);
        if (g.mode3d) {
          if (kc - L > 0) dmin = fmin(dmin, cz - (g.oz + (double)(kc - L) * g.sz));
          if (kc + L < nzm) dmin = fmin(dmin, (g.oz + (double)(kc + L + 1) * g.sz) - cz);
        }
        const double dm = dmin - eps;
        if (dm > 0.0 && kd < dm * dm) break;
      }
    }
    if ((uint32_t)lane < k) {
      idx_out[(uint64_t)qi * k + lane] = ri;
      if (d2_out) d2_out[(uint64_t)qi * k + lane] = rd;
    }
  }
}

// kNN query tiles (k <= KMAX, used for k <= kKnnTileMax): 32 cell-sorted
// centres per warp, one per
// lane, walk the hull of their Chebyshev-1 voxel blocks (3 x 3 x 3 around
// each centre's voxel) once — the radius tiles' staged, warp-uniform record
// stream — and each lane keeps its own sorted (d², handle) list of k in
// shared memory (stride 33). A lane is finished when the test the shell walk
// makes after shell 1 holds (list full and k-th d² below the squared
// distance to the nearest unvisited voxel face, or the block covers the
// grid); the shell walk would stop there with the same list, so the result
// is identical. Lanes that are not finished, and tiles whose hull exceeds 32
// columns, go to a redo list answered by knn_warp_kernel.
template <int KMAX>
struct KnnTileSmem {
  double d[KMAX * 33];
  uint32_t id[KMAX * 33];
  PointRec stg[64];
};

template <int FLAVOR, int KMAX>
__global__ void __launch_bounds__(kKThreads) knn_tile_kernel(
    const Tables t, const double* __restrict__ q, uint64_t nq, uint32_t k,
    const uint32_t* __restrict__ perm, uint32_t* __restrict__ idx_out,
    double* __restrict__ d2_out, uint32_t* __restrict__ redo, uint32_t* __restrict__ n_redo) {
  using namespace ::cmg::tw;
  extern __shared__ __align__(16) unsigned char ksm[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  KnnTileSmem<KMAX>& sm = reinterpret_cast<KnnTileSmem<KMAX>*>(ksm)[wib];
  double* ld = sm.d;
  uint32_t* li = sm.id;
  const DevGrid& g = t.g;
  const PointRec* __restrict__ rec = t.rec;
  const int64_t nx = (int64_t)g.nx, ny = (int64_t)g.ny, nzm = (int64_t)g.nz - 1;
  const uint64_t ntiles = (nq + 31) / 32;
  const uint64_t W = (uint64_t)gridDim.x * kKWarps;
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);
  for (uint64_t tile = (uint64_t)blockIdx.x * kKWarps + wib; tile < ntiles; tile += W) {
    const uint64_t s = tile * 32 + lane;
    const bool active = s < nq;
    const uint32_t qi = active ? __ldg(perm + s) : 0u;
    double cx = 0.0, cy = 0.0, cz = 0.0;
    if (active) {
      cx = __ldg(q + 3 * (uint64_t)qi);
      cy = __ldg(q + 3 * (uint64_t)qi + 1);
      cz = __ldg(q + 3 * (uint64_t)qi + 2);
    }
    const int64_t ic = (int64_t)axis_index(cx, g.ox, g.sx, g.nx);
    const int64_t jc = (int64_t)axis_index(cy, g.oy, g.sy, g.ny);
    const int64_t kc = g.mode3d ? (int64_t)axis_index(cz, g.oz, g.sz, g.nz) : 0;
    const int64_t i0 = imax64(0, ic - 1), i1 = imin64(nx - 1, ic + 1);
    const int64_t j0 = imax64(0, jc - 1), j1 = imin64(ny - 1, jc + 1);
    const int64_t k0 = imax64(0, kc - 1), k1 = imin64(nzm, kc + 1);
    const uint32_t I0 = warp_min_u32(active ? (uint32_t)i0 : 0xffffffffu);
    const uint32_t I1 = warp_max_u32(active ? (uint32_t)i1 : 0u);
    const uint32_t J0 = warp_min_u32(active ? (uint32_t)j0 : 0xffffffffu);
    const uint32_t J1 = warp_max_u32(active ? (uint32_t)j1 : 0u);
    const uint32_t K0 = warp_min_u32(active ? (uint32_t)k0 : 0xffffffffu);
    const uint32_t K1 = warp_max_u32(active ? (uint32_t)k1 : 0u);
    const uint32_t nj = J1 - J0 + 1;
    const uint64_t nc = (uint64_t)(I1 - I0 + 1) * nj;
    bool done = false;
    if (nc <= 32) {
      uint32_t b = 0, e = 0;
      if ((uint32_t)lane < nc)
        column_span<FLAVOR>(t, I0 + lane / nj, J0 + lane % nj, K0, K1, &b, &e);
      uint32_t colmask = 0;
      if (active) {
        const uint64_t rowbits = ((1ull << ((uint32_t)(j1 - j0) + 1)) - 1ull) << ((uint32_t)j0 - J0);
        for (uint32_t ci = (uint32_t)i0 - I0; ci <= (uint32_t)i1 - I0; ++ci)
          colmask |= (uint32_t)(rowbits << (ci * nj));
      }
      const uint32_t kk0 = (uint32_t)k0, kspan = (uint32_t)(k1 - k0);
      uint32_t needmask = colmask;
#pragma unroll
      for (int sh = 16; sh > 0; sh >>= 1) needmask |= __shfl_xor_sync(0xffffffffu, needmask, sh);
      needmask &= __ballot_sync(0xffffffffu, e > b);
      uint32_t cnt = 0;
      double kd = kInf;
      uint32_t kid = 0xffffffffu;
      uint32_t c = 0, p = 0, ce = 0;
      bool more = advance_chunk(needmask, c, p, ce, b, e, true);
      int buf = 0;
      if (more) stage_chunk(sm.stg, rec, p, min(32u, ce - p), lane);
      cp_async_commit();
      while (more) {
        uint32_t c2 = c, p2 = p, ce2 = ce;
        const bool more2 = advance_chunk(needmask, c2, p2, ce2, b, e, false);
        if (more2) stage_chunk(sm.stg + (buf ^ 1) * 32, rec, p2, min(32u, ce2 - p2), lane);
        cp_async_commit();
        cp_async_wait<1>();
        __syncwarp();
        const SRec* sr = reinterpret_cast<const SRec*>(sm.stg + buf * 32);
        const uint32_t len = min(32u, ce - p);
        const bool need = active && ((colmask >> c) & 1u);
        for (uint32_t u = 0; u < len; ++u) {
          const SRec v = sr[u];
          if (need && v.meta - kk0 <= kspan) {
            const double d2 = sqdist(v.x, v.y, v.z, cx, cy, cz);
            if (cnt < k || pair_less(d2, v.id, kd, kid)) {
              uint32_t pos = cnt < k ? cnt : k - 1;
              CM_DCHECK(pos < (uint32_t)KMAX);
              while (pos > 0) {
                const double pd = ld[(pos - 1) * 33 + lane];
                const uint32_t pi = li[(pos - 1) * 33 + lane];
                if (!pair_less(d2, v.id, pd, pi)) break;
                ld[pos * 33 + lane] = pd;
                li[pos * 33 + lane] = pi;
                --pos;
              }
              ld[pos * 33 + lane] = d2;
              li[pos * 33 + lane] = v.id;
              if (cnt < k) ++cnt;
              if (cnt == k) {
                kd = ld[(k - 1) * 33 + lane];
                kid = li[(k - 1) * 33 + lane];
              }
            }
          }
        }
        __syncwarp();
        buf ^= 1;
        c = c2, p = p2, ce = ce2;
        more = more2;
      }
      cp_async_wait<0>();
      // the shell walk's stop test after shell 1 (knn_warp_kernel)
      const bool all = i0 == 0 && i1 == nx - 1 && j0 == 0 && j1 == ny - 1 && k0 == 0 && k1 == nzm;
      if (all) {
        done = true;
      } else if (cnt == k) {
        const double eps = 1e-12 * (fabs(cx) + fabs(cy) + fabs(cz) + fabs(g.ox) + fabs(g.oy) +
                                    fabs(g.oz) + g.sx + g.sy + g.sz);
        double dmin = 1e300;
        if (i0 > 0) dmin = fmin(dmin, cx - (g.ox + (double)i0 * g.sx));
        if (i1 < nx - 1) dmin = fmin(dmin, (g.ox + (double)(i1 + 1) * g.sx) - cx);
        if (j0 > 0) dmin = fmin(dmin, cy - (g.oy + (double)j0 * g.sy));
        if (j1 < ny - 1) dmin = fmin(dmin, (g.oy + (double)(j1 + 1) * g.sy) - cy);
        if (g.mode3d) {
          if (k0 > 0) dmin = fmin(dmin, cz - (g.oz + (double)k0 * g.sz));
          if (k1 < nzm) dmin = fmin(dmin, (g.oz + (double)(k1 + 1) * g.sz) - cz);
        }
        const double dm = dmin - eps;
        done = dm > 0.0 && kd < dm * dm;
      }
      if (active && done) {
        for (uint32_t x = 0; x < k; ++x) {
          idx_out[(uint64_t)qi * k + x] = x < cnt ? li[x * 33 + lane] : 0xffffffffu;
          if (d2_out) d2_out[(uint64_t)qi * k + x] = x < cnt ? ld[x * 33 + lane] : kInf;
        }
      }
    }
    const uint32_t rm = __ballot_sync(0xffffffffu, active && !done);
    if (rm) {
      uint32_t slot = 0;
      if (lane == 0) slot = atomicAdd(n_redo, (uint32_t)__popc(rm));
      slot = __shfl_sync(0xffffffffu, slot, 0);
      if ((rm >> lane) & 1u) redo[slot + __popc(rm & lanemask_lt())] = qi;
    }
    __syncwarp();
  }
}

// ---- per-thread kNN (k <= 64, the default) --------------------------------
// One THREAD per centre (cell-sorted, so a warp's 32 centres are spatial
// neighbours and share their records through L1): the thread walks its own
// Chebyshev voxel shells — the 3 x 3 x 3 block first, own column first —
// keeping its k best (d², handle) in a max-heap in shared memory (entry e of
// thread t at [e][t], conflict-free), and stops with the shell walk's exact
// test. Against one warp per centre there are no per-centre span lookups or
// batch merges on the warp's critical path and no lanes idle on another
// centre's candidates. Pass 1 stops at shell LFIRST; the centres it cannot
// finish are compacted into a redo list and walked again, all shells, by a
// second launch (so hard centres share warps with hard centres).
constexpr int kTThreads = 128;

template <int K>
struct KnnHeap {
  double* d;
  uint32_t* id;
  __device__ __forceinline__ double dd(uint32_t e) const { return d[e * kTThreads]; }
  __device__ __forceinline__ uint32_t ii(uint32_t e) const { return id[e * kTThreads]; }
  __device__ __forceinline__ void put(uint32_t e, double x, uint32_t xi) {
    d[e * kTThreads] = x;
    id[e * kTThreads] = xi;
  }
  // max-heap of n entries by (d², handle): insert (n < cap)
  __device__ __forceinline__ void push(uint32_t n, double x, uint32_t xi) {
    uint32_t pos = n;
    while (pos > 0) {
      const uint32_t par = (pos - 1) >> 1;
      const double pd = dd(par);
      const uint32_t pi = ii(par);
      if (!pair_less(pd, pi, x, xi)) break;
      put(pos, pd, pi);
      pos = par;
    }
    put(pos, x, xi);
  }
  // replace the root (largest) by a smaller entry, heap of n
  __device__ __forceinline__ void replace_top(uint32_t n, double x, uint32_t xi) {
    uint32_t pos = 0;
    for (;;) {
      uint32_t c = 2 * pos + 1;
      if (c >= n) break;
      double cd = dd(c);
      uint32_t ci = ii(c);
      if (c + 1 < n) {
        const double rd = dd(c + 1);
        const uint32_t ri = ii(c + 1);
        if (pair_less(cd, ci, rd, ri)) cd = rd, ci = ri, ++c;
      }
      if (!pair_less(x, xi, cd, ci)) break;
      put(pos, cd, ci);
      pos = c;
    }
    put(pos, x, xi);
  }
};

// BALL: ball completion after the first full block (k > 16); otherwise
// whole shells with the stop test after each (fewer registers: measured
// faster at k = 8 / 16, 8.6 / 12.5 ms against 11.2 / 16.2 ms on config 3).
#ifndef CM_KNN_TBALL
#define CM_KNN_TBALL 1  // ball completion in the per-thread kernel for k > 16
#endif
template <int FLAVOR, int K, bool BALL = (CM_KNN_TBALL && K > 16)>
__global__ void __launch_bounds__(kTThreads, (K > 16 ? 4 : K > 8 ? CM_KNN_TMINB : CM_KNN_TMINB8)) knn_thread_kernel(
    const Tables t, const double* __restrict__ q, uint64_t nq, uint32_t k,
    const uint32_t* __restrict__ list, const uint32_t* __restrict__ n_list, int lmax,
    uint32_t* __restrict__ idx_out, double* __restrict__ d2_out, uint32_t* __restrict__ redo,
    uint32_t* __restrict__ n_redo, double r0) {
  extern __shared__ __align__(16) unsigned char hsm[];
  double* sd = reinterpret_cast<double*>(hsm);
  uint32_t* sid = reinterpret_cast<uint32_t*>(hsm + (size_t)K * kTThreads * sizeof(double));
  KnnHeap<K> h{sd + threadIdx.x, sid + threadIdx.x};
  if (n_list) nq = nq < (uint64_t)*n_list ? nq : (uint64_t)*n_list;
  const DevGrid& g = t.g;
  const PointRec* __restrict__ rec = t.rec;
  const int64_t nx = (int64_t)g.nx, ny = (int64_t)g.ny, nzm = (int64_t)g.nz - 1;
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);
  const uint64_t stride = (uint64_t)gridDim.x * kTThreads;
  for (uint64_t s0 = (uint64_t)blockIdx.x * kTThreads; s0 < nq; s0 += stride) {
    const uint64_t s = s0 + threadIdx.x;
    const bool active = s < nq;
    bool done = !active;
    uint32_t qi = 0, cnt = 0;
    if (active) {
      qi = __ldg(list + s);
      const double cx = __ldg(q + 3 * (uint64_t)qi);
      const double cy = __ldg(q + 3 * (uint64_t)qi + 1);
      const double cz = __ldg(q + 3 * (uint64_t)qi + 2);
      const int64_t ic = (int64_t)axis_index(cx, g.ox, g.sx, g.nx);
      const int64_t jc = (int64_t)axis_index(cy, g.oy, g.sy, g.ny);
      const int64_t kc = g.mode3d ? (int64_t)axis_index(cz, g.oz, g.sz, g.nz) : 0;
      const double eps = 1e-12 * (fabs(cx) + fabs(cy) + fabs(cz) + fabs(g.ox) + fabs(g.oy) +
                                  fabs(g.oz) + g.sx + g.sy + g.sz);
      double kd = kInf;       // the heap's root (k-th best) once full
      uint32_t kid = 0xffffffffu;
      auto offer = [&](double d2, uint32_t id) {
        if (cnt < k) {
          h.push(cnt, d2, id);
          if (++cnt == k) kd = h.dd(0), kid = h.ii(0);
        } else if (pair_less(d2, id, kd, kid)) {
          h.replace_top(k, d2, id);
          kd = h.dd(0), kid = h.ii(0);
        }
      };
      // records in groups of four: all four loads in flight before the
      // first distance is needed (the walk is load-latency bound otherwise).
      // (Screening candidates on the fp32 records first — filter.cuh — and
      // loading the fp64 record only for possible improvements measured
      // slower: config 3 k = 8 9.6 -> 13.2 ms.)
      auto visit = [&](uint32_t b, uint32_t e, int64_t, int64_t) {
        uint32_t p = b;
        constexpr int B = CM_KNN_TBATCH;
        for (; p + B <= e; p += B) {
          PointRec pr[B];
#pragma unroll
          for (int u = 0; u < B; ++u) pr[u] = load_rec(rec + p + u);
          double d2[B];
#pragma unroll
          for (int u = 0; u < B; ++u) d2[u] = sqdist(pr[u].x, pr[u].y, pr[u].z, cx, cy, cz);
#pragma unroll
          for (int u = 0; u < B; ++u) offer(d2[u], pr[u].id);
        }
        for (; p < e; ++p) {
          const PointRec pr = load_rec(rec + p);
          offer(sqdist(pr.x, pr.y, pr.z, cx, cy, cz), pr.id);
        }
      };
      // (1) the 3 x 3 x 3 block, own column first; (2) further Chebyshev
      // shells only while fewer than k points are known; (3) the shell
      // walk's stop test, and where it fails, ball completion: every voxel
      // of clamped_range(c +- R) outside the visited block, R = the current
      // k-th distance rounded up. A point that beats the final k-th has fp64
      // d² <= kd, so its true distance is <= sqrt(kd)(1 + 2^-51) <= R and it
      // lies in that voxel range (axis_index is monotone): exact, and a
      // centre visits only the voxels its k-th neighbour ball touches
      // instead of whole shells.
      if (CM_KNN_BOX && r0 > 0.0) {
        // Radius boxes: visit every voxel of clamped_range(c +- R) for R =
        // r0 (the expected k-th distance, from the cloud's mean density),
        // doubling R while fewer than k points are known; then ball
        // completion at the k-th distance. The visited set is always the
        // last box (boxes grow monotonically), so each step visits only the
        // new box minus the old one: per column the k ranges below and
        // above the old box, or the whole k range outside its (i, j) range.
        Range V{};
        bool hasV = false;
        auto visit_new = [&](const Range& B) {
          const int64_t bi0 = (int64_t)B.i0, bi1 = (int64_t)B.i1, bj0 = (int64_t)B.j0,
                        bj1 = (int64_t)B.j1;
          const int64_t nbj = bj1 - bj0 + 1, nbc = (bi1 - bi0 + 1) * nbj;
          const bool own = ic >= bi0 && ic <= bi1 && jc >= bj0 && jc <= bj1;
          for (int64_t c = -1; c < nbc; ++c) {
            int64_t i, j;
            if (c < 0) {  // the centre's own column first: a tight k-th early
              if (!own) continue;
              i = ic, j = jc;
            } else {
              i = bi0 + c / nbj, j = bj0 + c % nbj;
              if (own && i == ic && j == jc) continue;
            }
            const bool inV = hasV && i >= (int64_t)V.i0 && i <= (int64_t)V.i1 &&
                             j >= (int64_t)V.j0 && j <= (int64_t)V.j1;
            int64_t lo1 = (int64_t)B.k0, hi1 = (int64_t)B.k1, lo2 = 1, hi2 = 0;
            if (inV) {
              hi1 = imin64(hi1, (int64_t)V.k0 - 1);
              lo2 = imax64((int64_t)B.k0, (int64_t)V.k1 + 1);
              hi2 = (int64_t)B.k1;
            }
            uint32_t b, e;
            if (lo1 <= hi1) {
              column_span<FLAVOR>(t, (uint64_t)i, (uint64_t)j, (uint64_t)lo1, (uint64_t)hi1, &b, &e);
              visit(b, e, i, j);
            }
            if (lo2 <= hi2) {
              column_span<FLAVOR>(t, (uint64_t)i, (uint64_t)j, (uint64_t)lo2, (uint64_t)hi2, &b, &e);
              visit(b, e, i, j);
            }
          }
        };
        auto merge_box = [&](const Range& B) {
          if (!hasV) {
            V = B;
            hasV = true;
            return;
          }
          V.i0 = min(V.i0, B.i0), V.i1 = max(V.i1, B.i1);
          V.j0 = min(V.j0, B.j0), V.j1 = max(V.j1, B.j1);
          V.k0 = min(V.k0, B.k0), V.k1 = max(V.k1, B.k1);
        };
        double R = r0;
        for (;;) {
          Range B;
          if (clamped_range(g, cx, cy, cz, R, &B, 0)) {
            visit_new(B);
            merge_box(B);
          }
          if (cnt >= k) break;
          if (hasV && V.i0 == 0 && V.i1 == (uint64_t)(nx - 1) && V.j0 == 0 &&
              V.j1 == (uint64_t)(ny - 1) && V.k0 == 0 && V.k1 == (uint64_t)nzm)
            break;  // the whole grid: fewer than k points
          R *= 2.0;
        }
        if (cnt == k) {
          Range B;
          const double Rk = sqrt(kd) * (1.0 + 1e-12) + eps;
          if (clamped_range(g, cx, cy, cz, Rk, &B, 0)) visit_new(B);
        }
        done = true;
      } else {
      int64_t L = 1;
      bool all = false;
      for (;; ++L) {
        const int64_t i0 = imax64(0, ic - L), i1 = imin64(nx - 1, ic + L);
        const int64_t j0 = imax64(0, jc - L), j1 = imin64(ny - 1, jc + L);
        const int64_t nj = j1 - j0 + 1;
        const int64_t ncol = (i1 - i0 + 1) * nj;
        if (CM_KNN_PRUNE && L == 1) {
          // The 3 x 3 x 3 block with pruning: once k points are known, a
          // neighbour column (and each of its three voxels) is skipped when
          // every point it can hold is farther than the current k-th: the
          // squared distance from the centre to the column's (voxel's) near
          // faces, each face distance reduced by the stop test's rounding
          // margin, strictly exceeds the k-th d². The k-th only shrinks, so
          // a skipped point can never enter the result: exact.
          uint32_t b, e;
          column_span<FLAVOR>(t, (uint64_t)ic, (uint64_t)jc, (uint64_t)imax64(0, kc - 1),
                              (uint64_t)imin64(nzm, kc + 1), &b, &e);
          visit(b, e, ic, jc);
          // lower bounds of |dx| to the columns at ic -/+ 1 (same for y, z)
          const double fxm = fmax(0.0, (cx - (g.ox + (double)ic * g.sx)) - eps);
          const double fxp = fmax(0.0, ((g.ox + (double)(ic + 1) * g.sx) - cx) - eps);
          const double fym = fmax(0.0, (cy - (g.oy + (double)jc * g.sy)) - eps);
          const double fyp = fmax(0.0, ((g.oy + (double)(jc + 1) * g.sy) - cy) - eps);
          const double fzm = fmax(0.0, (cz - (g.oz + (double)kc * g.sz)) - eps);
          const double fzp = fmax(0.0, ((g.oz + (double)(kc + 1) * g.sz) - cz) - eps);
          // CM_KNN_PRUNE == 2: nearest columns first, relative to each centre
          // (near x side, near y side, near corner, far sides, far corners)
          const int nsx = (CM_KNN_PRUNE == 2 && fxp < fxm) ? 1 : -1;
          const int nsy = (CM_KNN_PRUNE == 2 && fyp < fym) ? 1 : -1;
#pragma unroll 1
          for (int c = 0; c < 8; ++c) {
            int di, dj;
            if (CM_KNN_PRUNE == 2) {
              di = ((int)((0x926u >> (2 * c)) & 3u) - 1) * nsx;
              dj = ((int)((0x2069u >> (2 * c)) & 3u) - 1) * nsy;
            } else {
              const int cc = c + (c >= 4);  // 0..8 without the centre (4)
              di = cc / 3 - 1, dj = cc % 3 - 1;
            }
            const int64_t i = ic + di, j = jc + dj;
            if (i < 0 || i >= nx || j < 0 || j >= ny) continue;
            int64_t klo = imax64(0, kc - 1), khi = imin64(nzm, kc + 1);
            if (cnt == k) {
              const double bx = di == 0 ? 0.0 : (di < 0 ? fxm : fxp);
              const double by = dj == 0 ? 0.0 : (dj < 0 ? fym : fyp);
              const double lb2 = bx * bx + by * by;
              if (kd < lb2) continue;
              if (g.mode3d) {
                if (kd < lb2 + fzm * fzm) klo = kc;
                if (kd < lb2 + fzp * fzp) khi = kc;
              }
            }
            column_span<FLAVOR>(t, (uint64_t)i, (uint64_t)j, (uint64_t)klo, (uint64_t)khi, &b, &e);
            visit(b, e, i, j);
          }
        } else
        for (int64_t c = -1; c < ncol; ++c) {
          int64_t i, j;
          if (c < 0) {
            if (L != 1) continue;
            i = ic, j = jc;
          } else {
            i = i0 + c / nj, j = j0 + c % nj;
            if (L == 1 && i == ic && j == jc) continue;
          }
          const bool ring = L == 1 || i == ic - L || i == ic + L || j == jc - L || j == jc + L;
          uint32_t b1, e1, b2, e2;
          shell_column_spans<FLAVOR>(t, i, j, ring, kc, L, (uint64_t)nzm, &b1, &e1, &b2, &e2);
          visit(b1, e1, i, j);
          visit(b2, e2, i, j);
        }
        all = i0 == 0 && i1 == nx - 1 && j0 == 0 && j1 == ny - 1 && imax64(0, kc - L) == 0 &&
              imin64(nzm, kc + L) == nzm;
        if (all) break;
        if (cnt == k) {
          if (BALL) break;  // the stop test and ball completion follow
          // without ball completion: the shell walk's stop test, every shell
          const int64_t si0 = imax64(0, ic - L), si1 = imin64(nx - 1, ic + L);
          const int64_t sj0 = imax64(0, jc - L), sj1 = imin64(ny - 1, jc + L);
          double dmin = 1e300;
          if (si0 > 0) dmin = fmin(dmin, cx - (g.ox + (double)si0 * g.sx));
          if (si1 < nx - 1) dmin = fmin(dmin, (g.ox + (double)(si1 + 1) * g.sx) - cx);
          if (sj0 > 0) dmin = fmin(dmin, cy - (g.oy + (double)sj0 * g.sy));
          if (sj1 < ny - 1) dmin = fmin(dmin, (g.oy + (double)(sj1 + 1) * g.sy) - cy);
          if (g.mode3d) {
            if (kc - L > 0) dmin = fmin(dmin, cz - (g.oz + (double)(kc - L) * g.sz));
            if (kc + L < nzm) dmin = fmin(dmin, (g.oz + (double)(kc + L + 1) * g.sz) - cz);
          }
          const double dm = dmin - eps;
          if (dm > 0.0 && kd < dm * dm) {
            all = true;
            break;
          }
        }
        if (L >= lmax) break;
      }
      if (BALL && cnt == k && !all) {
        const int64_t i0 = imax64(0, ic - L), i1 = imin64(nx - 1, ic + L);
        const int64_t j0 = imax64(0, jc - L), j1 = imin64(ny - 1, jc + L);
        double dmin = 1e300;
        if (i0 > 0) dmin = fmin(dmin, cx - (g.ox + (double)i0 * g.sx));
        if (i1 < nx - 1) dmin = fmin(dmin, (g.ox + (double)(i1 + 1) * g.sx) - cx);
        if (j0 > 0) dmin = fmin(dmin, cy - (g.oy + (double)j0 * g.sy));
        if (j1 < ny - 1) dmin = fmin(dmin, (g.oy + (double)(j1 + 1) * g.sy) - cy);
        if (g.mode3d) {
          if (kc - L > 0) dmin = fmin(dmin, cz - (g.oz + (double)(kc - L) * g.sz));
          if (kc + L < nzm) dmin = fmin(dmin, (g.oz + (double)(kc + L + 1) * g.sz) - cz);
        }
        const double dm = dmin - eps;
        if (dm > 0.0 && kd < dm * dm) all = true;  // nothing unvisited can beat the k-th
      }
      if (BALL && cnt == k && !all) {
        const double R = sqrt(kd) * (1.0 + 1e-12) + eps;
        Range B;
        if (clamped_range(g, cx, cy, cz, R, &B, 0)) {
          for (int64_t i = (int64_t)B.i0; i <= (int64_t)B.i1; ++i)
            for (int64_t j = (int64_t)B.j0; j <= (int64_t)B.j1; ++j) {
              const bool inblock = i >= ic - L && i <= ic + L && j >= jc - L && j <= jc + L;
              int64_t lo1 = (int64_t)B.k0, hi1 = (int64_t)B.k1, lo2 = 1, hi2 = 0;
              if (inblock) {  // only the parts below and above the block
                hi1 = imin64(hi1, kc - L - 1);
                lo2 = imax64((int64_t)B.k0, kc + L + 1);
                hi2 = (int64_t)B.k1;
              }
              uint32_t b, e;
              if (lo1 <= hi1) {
                column_span<FLAVOR>(t, (uint64_t)i, (uint64_t)j, (uint64_t)lo1, (uint64_t)hi1, &b, &e);
                visit(b, e, i, j);
              }
              if (lo2 <= hi2) {
                column_span<FLAVOR>(t, (uint64_t)i, (uint64_t)j, (uint64_t)lo2, (uint64_t)hi2, &b, &e);
                visit(b, e, i, j);
              }
            }
        }
        done = true;
      } else if (all) {
        done = true;  // fewer than k points in the whole grid, or the stop test holds
      }
      }
      if (done) {
        // heapsort in place: ascending (d², handle)
        for (uint32_t n = cnt; n > 1; --n) {
          const double td = h.dd(0);
          const uint32_t ti = h.ii(0);
          const double xd = h.dd(n - 1);
          const uint32_t xi = h.ii(n - 1);
          h.put(n - 1, td, ti);
          h.replace_top(n - 1, xd, xi);
        }
        for (uint32_t x = 0; x < k; ++x) {
          idx_out[(uint64_t)qi * k + x] = x < cnt ? h.ii(x) : 0xffffffffu;
          if (d2_out) d2_out[(uint64_t)qi * k + x] = x < cnt ? h.dd(x) : kInf;
        }
      }
    }
    const bool r = active && !done;
    const uint32_t rm = __ballot_sync(0xffffffffu, r);
    if (rm) {
      const int lane = threadIdx.x & 31;
      uint32_t slot = 0;
      if (lane == __ffs(rm) - 1) slot = atomicAdd(n_redo, (uint32_t)__popc(rm));
      slot = __shfl_sync(0xffffffffu, slot, __ffs(rm) - 1);
      if (r) redo[slot + __popc(rm & lanemask_lt())] = qi;
    }
  }
}

// ---- kNN by radius brackets (opt-in) ---------------------------------------
// The k nearest of a centre are exactly the k smallest (d², handle) among
// the points with d² <= R² for ANY R with count(d² <= R²) >= k. So: (1)
// per-centre radius brackets from the radius engine's COUNT pass (the same
// query tiles: 32 cell-sorted centres share each staged record), growing R
// for the centres that saw fewer than k points; (2) one COLLECT pass at each
// centre's final R (its hits land in an arena row); (3) each row sorted by
// (d², handle) and cut to k. Centres still open after the last bracket, or
// with rows too long to sort in registers, take the shell walk above.
constexpr int kSelMax = 512;  // longest row sorted by knn_select_kernel

// Round outcome of list entry s: 0 resolved (count in [k, kSelMax]), 1 grow
// the radius and retry, 2 shell walk (last round, or the row is too long).
__global__ void knn_bracket_kernel(const uint32_t* __restrict__ list, uint32_t n,
                                   const uint32_t* __restrict__ counts, uint32_t k, int last,
                                   double* __restrict__ rq, uint32_t* __restrict__ f_res,
                                   uint32_t* __restrict__ f_next, double rmax) {
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < n; s += gridDim.x * blockDim.x) {
    const uint32_t qi = list[s];
    const uint32_t c = counts[qi];
    const double r = rq[qi];
    uint32_t res = 0, nxt = 0;
    if (c >= k && c <= (uint32_t)kSelMax) {
      res = 1;
    } else if (c < k && !last && r < rmax) {
      // grow as for a surface (count ~ r^2), by 1.25..2x, 5 % margin
      const double g = fmin(2.0, fmax(1.25, 1.05 * sqrt((double)k / fmax(1.0, (double)c))));
      rq[qi] = r * g;
      nxt = 1;
    }
    f_res[s] = res;
    f_next[s] = nxt;
  }
}

// Order-preserving compaction of the round: resolved entries are appended
// after the earlier rounds' (res_base), retries form the next list, the rest
// go to the shell-walk list (any order).
__global__ void knn_compact_kernel(const uint32_t* __restrict__ list, uint32_t n,
                                   const uint32_t* __restrict__ f_res, const uint32_t* __restrict__ p_res,
                                   const uint32_t* __restrict__ f_next, const uint32_t* __restrict__ p_next,
                                   uint32_t* __restrict__ res_list, const uint32_t* __restrict__ res_base,
                                   uint32_t* __restrict__ next_list, uint32_t* __restrict__ walk_list,
                                   uint32_t* __restrict__ n_walk) {
  const uint32_t rb = *res_base;
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < n; s += gridDim.x * blockDim.x) {
    const uint32_t qi = list[s];
    if (f_res[s]) res_list[rb + p_res[s]] = qi;
    else if (f_next[s]) next_list[p_next[s]] = qi;
    else walk_list[atomicAdd(n_walk, 1u)] = qi;
  }
}

__global__ void knn_rank_kernel(const PointRec* __restrict__ rec, uint64_t n,
                                uint32_t* __restrict__ rec_of) {
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < n;
       p += (uint64_t)gridDim.x * blockDim.x)
    rec_of[rec[p].id] = (uint32_t)p;
}

// Bitonic sort of 32 * E (d², handle) pairs held blocked by a warp (lane l:
// elements [l * E, (l + 1) * E)), ascending by (d², handle).
template <int E>
__device__ __forceinline__ void warp_sort_pairs_blocked(double (&d)[E], uint32_t (&id)[E], int lane) {
  constexpr int P = 32 * E;
#pragma unroll
  for (int kk = 2; kk <= P; kk <<= 1) {
#pragma unroll
    for (int j = kk >> 1; j > 0; j >>= 1) {
      if (j < E) {
#pragma unroll
        for (int r = 0; r < E; ++r) {
          const int p = r ^ j;
          if (p > r) {
            const bool asc = (((uint32_t)lane * E + r) & kk) == 0;
            const bool pl = pair_less(d[p], id[p], d[r], id[r]);
            if (asc == pl) {
              const double td = d[r];
              d[r] = d[p];
              d[p] = td;
              const uint32_t ti = id[r];
              id[r] = id[p];
              id[p] = ti;
            }
          }
        }
      } else {
        const int jl = j / E;
        const bool lower = (lane & jl) == 0;
#pragma unroll
        for (int r = 0; r < E; ++r) {
          const double od = __shfl_xor_sync(0xffffffffu, d[r], jl);
          const uint32_t oi = __shfl_xor_sync(0xffffffffu, id[r], jl);
          const bool asc = (((uint32_t)lane * E + r) & kk) == 0;
          const bool o_less = pair_less(od, oi, d[r], id[r]);
          if ((lower == asc) ? o_less : !o_less) {
            d[r] = od;
            id[r] = oi;
          }
        }
      }
    }
  }
}

// ---- kNN by histogram selection (16 < k <= 64) -----------------------------
// One warp per centre. For the Chebyshev block L around the centre's voxel
// (L = 1, 2, ...: one span lookup per column, lanes = columns), D = the
// squared distance to the nearest unvisited voxel face (the shell walk's stop
// bound). Pass A walks the block's candidates (32 per step, coalesced) and
// counts the ones with d² < D in 32 bins uniform in d²; if at least k lie
// below D, the bin b* that holds the k-th is known, and pass B walks the same
// spans again and keeps every candidate with bin <= b* (bins are monotone in
// d², so these are a prefix of the candidates in (d², handle) order that
// holds the k best; all of them lie below D, so the shell walk's stop test
// holds and the block's k best are the answer). The kept ones (k .. 128) are
// sorted once in registers: no per-candidate list maintenance. Centres whose block never holds k points below D within
// lmax levels, whose bin b* overflows the buffer (heavy ties), or whose
// block covers the whole grid go to the redo list (shell walk).
constexpr int kHistCap = 128;

// The same network with the merge and cross-lane loops ROLLED (exchange
// distances and directions at run time; only the in-lane steps are
// unrolled): a fifth of the code. The unrolled E = 4 network did not fit the
// instruction cache next to the histogram kernel's walk (no_inst on half of
// its stall samples at k = 64).
template <int E>
__device__ __forceinline__ void warp_sort_pairs_blocked_rolled(double (&d)[E], uint32_t (&id)[E],
                                                               int lane) {
  constexpr int P = 32 * E;
#pragma unroll 1
  for (int kk = 2; kk <= P; kk <<= 1) {
#pragma unroll 1
    for (int j = kk >> 1; j >= E; j >>= 1) {
      const int jl = j / E;
      const bool lower = (lane & jl) == 0;
#pragma unroll
      for (int r = 0; r < E; ++r) {
        const double od = __shfl_xor_sync(0xffffffffu, d[r], jl);
        const uint32_t oi = __shfl_xor_sync(0xffffffffu, id[r], jl);
        const bool asc = (((uint32_t)lane * E + r) & kk) == 0;
        const bool o_less = pair_less(od, oi, d[r], id[r]);
        if ((lower == asc) ? o_less : !o_less) {
          d[r] = od;
          id[r] = oi;
        }
      }
    }
#pragma unroll
    for (int j = E >> 1; j > 0; j >>= 1) {
      if (j < kk) {
#pragma unroll
        for (int r = 0; r < E; ++r) {
          const int p = r ^ j;
          if (p > r) {
            const bool asc = (((uint32_t)lane * E + r) & kk) == 0;
            const bool pl = pair_less(d[p], id[p], d[r], id[r]);
            if (asc == pl) {
              const double td = d[r];
              d[r] = d[p];
              d[p] = td;
              const uint32_t ti = id[r];
              id[r] = id[p];
              id[p] = ti;
            }
          }
        }
      }
    }
  }
}

#ifndef CM_KNN_HIST_ROLLED
#define CM_KNN_HIST_ROLLED 1
#endif
template <int E>
__device__ __forceinline__ void hist_sort_out(const double* __restrict__ bd,
                                              const uint32_t* __restrict__ bi, uint32_t m,
                                              uint32_t k, uint64_t qi, int lane,
                                              uint32_t* __restrict__ idx_out,
                                              double* __restrict__ d2_out) {
  double d[E];
  uint32_t id[E];
#pragma unroll
  for (int r = 0; r < E; ++r) {
    const uint32_t i = (uint32_t)lane * E + r;
    d[r] = i < m ? bd[i] : __longlong_as_double(0x7ff0000000000000ll);
    id[r] = i < m ? bi[i] : 0xffffffffu;
  }
  if (CM_KNN_HIST_ROLLED && E >= 4) warp_sort_pairs_blocked_rolled<E>(d, id, lane);  // k = 64: 33.1 -> 32.2 ms; E = 2 (k = 40) is faster unrolled
  else warp_sort_pairs_blocked<E>(d, id, lane);
#pragma unroll
  for (int r = 0; r < E; ++r) {
    const uint32_t i = (uint32_t)lane * E + r;
    if (i < k) {
      idx_out[qi * k + i] = id[r];
      if (d2_out) d2_out[qi * k + i] = d[r];
    }
  }
}

__device__ __forceinline__ int hist_bin(double d2, double scale) {
  const int b = (int)__dmul_rn(d2, scale);
  return b > 31 ? 31 : b;
}

#ifndef CM_KNN_HIST_SKIP
#define CM_KNN_HIST_SKIP 1
#endif
#ifndef CM_KNN_HIST_MINB
#define CM_KNN_HIST_MINB 10  // 48 registers, small spill: config 3 k = 64 35.5 -> 33.7 ms
#endif
template <int FLAVOR>
__global__ void __launch_bounds__(kKThreads, CM_KNN_HIST_MINB) knn_hist_kernel(
    const Tables t, const double* __restrict__ q, uint64_t nq, uint32_t k,
    const uint32_t* __restrict__ perm, uint32_t* __restrict__ idx_out, double* __restrict__ d2_out,
    uint32_t* __restrict__ redo, uint32_t* __restrict__ n_redo, int lmax) {
  __shared__ uint32_t s_hist[kKWarps][32];
  __shared__ double s_bd[kKWarps][kHistCap];
  __shared__ uint32_t s_bi[kKWarps][kHistCap];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  uint32_t* hist = s_hist[wib];
  double* bd = s_bd[wib];
  uint32_t* bi = s_bi[wib];
  const uint64_t W = (uint64_t)gridDim.x * kKWarps;
  const DevGrid& g = t.g;
  const uint32_t lt = lanemask_lt();
  const int64_t nx = (int64_t)g.nx, ny = (int64_t)g.ny, nzm = (int64_t)g.nz - 1;
  for (uint64_t s = (uint64_t)blockIdx.x * kKWarps + wib; s < nq; s += W) {
    const uint32_t qi = perm ? __ldg(perm + s) : (uint32_t)s;
    const double cx = __ldg(q + 3 * (uint64_t)qi);
    const double cy = __ldg(q + 3 * (uint64_t)qi + 1);
    const double cz = __ldg(q + 3 * (uint64_t)qi + 2);
    const int64_t ic = (int64_t)axis_index(cx, g.ox, g.sx, g.nx);
    const int64_t jc = (int64_t)axis_index(cy, g.oy, g.sy, g.ny);
    const int64_t kc = g.mode3d ? (int64_t)axis_index(cz, g.oz, g.sz, g.nz) : 0;
    const double eps = 1e-12 * (fabs(cx) + fabs(cy) + fabs(cz) + fabs(g.ox) + fabs(g.oy) +
                                fabs(g.oz) + g.sx + g.sy + g.sz);
    bool finished = false;
    for (int64_t L = 1; L <= (int64_t)lmax; ++L) {
      const int64_t i0 = imax64(0, ic - L), i1 = imin64(nx - 1, ic + L);
      const int64_t j0 = imax64(0, jc - L), j1 = imin64(ny - 1, jc + L);
      const int64_t k0 = imax64(0, kc - L), k1 = imin64(nzm, kc + L);
      double dmin = 1e300;
      if (i0 > 0) dmin = fmin(dmin, cx - (g.ox + (double)i0 * g.sx));
      if (i1 < nx - 1) dmin = fmin(dmin, (g.ox + (double)(i1 + 1) * g.sx) - cx);
      if (j0 > 0) dmin = fmin(dmin, cy - (g.oy + (double)j0 * g.sy));
      if (j1 < ny - 1) dmin = fmin(dmin, (g.oy + (double)(j1 + 1) * g.sy) - cy);
      if (g.mode3d) {
        if (k0 > 0) dmin = fmin(dmin, cz - (g.oz + (double)k0 * g.sz));
        if (k1 < nzm) dmin = fmin(dmin, (g.oz + (double)(k1 + 1) * g.sz) - cz);
      }
      if (dmin == 1e300) break;  // the block is the whole grid: no bound, shell walk
      const double dm = dmin - eps;
      if (!(dm > 0.0)) continue;
      const double D = dm * dm;
      const double scale = 32.0 / D;
      const uint32_t nj = (uint32_t)(j1 - j0 + 1);
      const uint32_t ncol = (uint32_t)(i1 - i0 + 1) * nj;
      const bool single = ncol <= 32;
      uint32_t b = 0, len = 0, incl = 0, total = 0;
      int bstar = 0;
      uint32_t m = 0, pos = 0;
      bool ok = true;
      hist[lane] = 0;
      __syncwarp();
      for (int pass = 0; pass < 2 && ok; ++pass) {
        for (uint32_t cb = 0; cb < ncol; cb += 32) {
          if (pass == 0 || !single) {
            const uint32_t c = cb + lane;
            uint32_t e = 0;
            b = 0;
            if (c < ncol)
              column_span<FLAVOR>(t, (uint64_t)(i0 + (int64_t)(c / nj)), (uint64_t)(j0 + (int64_t)(c % nj)),
                                  (uint64_t)k0, (uint64_t)k1, &b, &e);
            len = e - b;
            incl = warp_incl_scan(len);
            total = __shfl_sync(0xffffffffu, incl, 31);
          }
          const uint32_t excl = incl - len;
          for (uint32_t t0 = 0; t0 < total; t0 += 32) {
            const uint32_t tt = t0 + lane;
            int Lq = 0;
#pragma unroll
            for (int sft = 16; sft > 0; sft >>= 1) {
              const uint32_t v = __shfl_sync(0xffffffffu, incl, Lq + sft - 1);
              if (v <= tt) Lq += sft;
            }
            const uint32_t xL = __shfl_sync(0xffffffffu, excl, Lq);
            const uint32_t bL = __shfl_sync(0xffffffffu, b, Lq);
            double d2 = 0.0;
            uint32_t id = 0;
            int bin = 32;
            if (tt < total) {
              const PointRec pr = load_rec(t.rec + bL + (tt - xL));
              d2 = sqdist(pr.x, pr.y, pr.z, cx, cy, cz);
              id = pr.id;
              if (d2 < D) bin = hist_bin(d2, scale);
            }
            if (pass == 0) {
              if (bin < 32) atomicAdd(hist + bin, 1u);
            } else {
              const bool sel = bin <= bstar;
              const uint32_t mm = __ballot_sync(0xffffffffu, sel);
              if (sel) {
                const uint32_t p = pos + __popc(mm & lt);
                CM_DCHECK(p < (uint32_t)kHistCap);
                bd[p] = d2;
                bi[p] = id;
              }
              pos += __popc(mm);
            }
          }
        }
        __syncwarp();
        if (pass == 0) {
          const uint32_t hi = warp_incl_scan(hist[lane]);
          const uint32_t ge = __ballot_sync(0xffffffffu, hi >= k);
          if (!ge) {
            ok = false;  // fewer than k below D: next level
            // far fewer than k (sparse neighbourhood): skip a level
            if (CM_KNN_HIST_SKIP && __shfl_sync(0xffffffffu, hi, 31) * 4u < k && L + 2 <= (int64_t)lmax) ++L;
          } else {
            bstar = __ffs(ge) - 1;
            m = __shfl_sync(0xffffffffu, hi, bstar);
            if (m > (uint32_t)kHistCap) ok = false, L = (int64_t)lmax;  // heavy bin: shell walk
          }
        }
      }
      if (!ok) continue;
      CM_DCHECK(pos == m);
      if (m <= 32) hist_sort_out<1>(bd, bi, m, k, (uint64_t)qi, lane, idx_out, d2_out);
      else if (m <= 64) hist_sort_out<2>(bd, bi, m, k, (uint64_t)qi, lane, idx_out, d2_out);
      else hist_sort_out<4>(bd, bi, m, k, (uint64_t)qi, lane, idx_out, d2_out);
      __syncwarp();
      finished = true;
      break;
    }
    if (!finished && lane == 0) redo[atomicAdd(n_redo, 1u)] = qi;
  }
}

template <int E>
__device__ __forceinline__ void select_row(const PointRec* __restrict__ rec,
                                           const uint32_t* __restrict__ rec_of,
                                           const uint32_t* __restrict__ row, uint32_t n, double cx,
                                           double cy, double cz, uint32_t k, uint64_t qi, int lane,
                                           uint32_t* __restrict__ idx_out,
                                           double* __restrict__ d2_out) {
  double d[E];
  uint32_t id[E];
#pragma unroll
  for (int r = 0; r < E; ++r) {
    const uint32_t i = (uint32_t)lane * E + r;
    d[r] = __longlong_as_double(0x7ff0000000000000ll);
    id[r] = 0xffffffffu;
    if (i < n) {
      const uint32_t h = __ldg(row + i);
      const PointRec pr = load_rec(rec + __ldg(rec_of + h));
      d[r] = sqdist(pr.x, pr.y, pr.z, cx, cy, cz);
      id[r] = h;
    }
  }
  warp_sort_pairs_blocked<E>(d, id, lane);
#pragma unroll
  for (int r = 0; r < E; ++r) {
    const uint32_t i = (uint32_t)lane * E + r;
    if (i < k) {
      idx_out[qi * k + i] = id[r];
      if (d2_out) d2_out[qi * k + i] = d[r];
    }
  }
}

// One warp per resolved centre: its arena row (every point with d² <= R²,
// at least k of them) sorted by (d², handle); the first k are the answer.
__global__ void __launch_bounds__(kKThreads) knn_select_kernel(
    const PointRec* __restrict__ rec, const uint32_t* __restrict__ rec_of,
    const double* __restrict__ q, const uint32_t* __restrict__ list,
    const uint32_t* __restrict__ n_list, uint32_t k, const uint32_t* __restrict__ arena,
    const uint64_t* __restrict__ toff, const uint32_t* __restrict__ scnt,
    uint32_t* __restrict__ idx_out, double* __restrict__ d2_out) {
  const int lane = threadIdx.x & 31;
  const uint32_t nl = *n_list;
  for (uint32_t s = blockIdx.x * kKWarps + (threadIdx.x >> 5); s < nl; s += gridDim.x * kKWarps) {
    const uint32_t qi = __ldg(list + s);
    const uint32_t n = __ldg(scnt + qi);
    const uint32_t* row = arena + __ldg(toff + qi);
    const double cx = __ldg(q + 3 * (uint64_t)qi);
    const double cy = __ldg(q + 3 * (uint64_t)qi + 1);
    const double cz = __ldg(q + 3 * (uint64_t)qi + 2);
    CM_DCHECK(n >= k && n <= (uint32_t)kSelMax);
    if (n <= 32)
      select_row<1>(rec, rec_of, row, n, cx, cy, cz, k, qi, lane, idx_out, d2_out);
    else if (n <= 64)
      select_row<2>(rec, rec_of, row, n, cx, cy, cz, k, qi, lane, idx_out, d2_out);
    else if (n <= 128)
      select_row<4>(rec, rec_of, row, n, cx, cy, cz, k, qi, lane, idx_out, d2_out);
    else if (n <= 256)
      select_row<8>(rec, rec_of, row, n, cx, cy, cz, k, qi, lane, idx_out, d2_out);
    else
      select_row<16>(rec, rec_of, row, n, cx, cy, cz, k, qi, lane, idx_out, d2_out);
  }
}

__global__ void fill_f64_kernel(double* __restrict__ a, uint64_t n, double v) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    a[i] = v;
}

__global__ void add_total_kernel(uint32_t* __restrict__ acc, const uint32_t* __restrict__ v) {
  *acc += *v;
}

// sum of counts over the resolved list -> *out (arena size)
__global__ void sum_counts_kernel(const uint32_t* __restrict__ list, const uint32_t* __restrict__ n_list,
                                  const uint32_t* __restrict__ counts,
                                  unsigned long long* __restrict__ out) {
  unsigned long long a = 0;
  const uint32_t n = *n_list;
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < n; s += gridDim.x * blockDim.x)
    a += counts[list[s]];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
  if ((threadIdx.x & 31) == 0 && a) atomicAdd(out, a);
}

unsigned kgrid(uint64_t n) {
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, (uint64_t)sm_count() * 8));
}

// The radius-bracket path (see knn_bracket_kernel). Centres it cannot finish
// go to walk[0 .. *n_walk) for the shell walk.
cm_status knn_brackets(const cm_index* ix, const double* q, uint64_t nq, uint32_t k,
                       const uint32_t* perm, uint32_t* idx, double* d2, cudaStream_t st,
                       uint32_t* walk, uint32_t* n_walk) {
  std::vector<void*> bufs;
  struct Free {
    std::vector<void*>& b;
    cudaStream_t st;
    ~Free() {
      for (void* p : b) dev_free(p, st);
    }
  } fr{bufs, st};
  auto alloc = [&](auto** p, size_t count) -> bool {
    if (dev_alloc_t(p, count, st) != cudaSuccess) return false;
    bufs.push_back(*p);
    return true;
  };
  const uint32_t* rec_of = nullptr;
  {
    std::lock_guard<std::mutex> lk(ix->lazy_mu);
    if (!ix->rec_of) {
      uint32_t* ro = nullptr;
      CM_CUDA_TRY(dev_alloc_t(&ro, ix->n, st));
      knn_rank_kernel<<<kgrid(ix->n), 256, 0, st>>>(ix->rec, ix->n, ro); ::cmg::note_launch();
      CM_CUDA_TRY(cudaGetLastError());
      ix->rec_of = ro;
    }
    rec_of = ix->rec_of;
  }
  double* rq = nullptr;
  uint32_t *counts = nullptr, *la = nullptr, *lb = nullptr, *res = nullptr, *f_res = nullptr,
           *f_next = nullptr, *p_res = nullptr, *p_next = nullptr, *part = nullptr,
           *n_res = nullptr, *scnt = nullptr;
  uint64_t* toff = nullptr;
  unsigned long long *cursor = nullptr, *cap_d = nullptr;
  if (!alloc(&rq, nq) || !alloc(&counts, nq + 1) || !alloc(&la, nq) || !alloc(&lb, nq) ||
      !alloc(&res, nq) || !alloc(&f_res, nq + 1) || !alloc(&f_next, nq + 1) ||
      !alloc(&p_res, nq + 1) || !alloc(&p_next, nq + 1) || !alloc(&part, scan_part_elems(nq)) ||
      !alloc(&n_res, 1) || !alloc(&scnt, nq + 1) || !alloc(&toff, nq + 1) || !alloc(&cursor, 2) ||
      !alloc(&cap_d, 1)) {
    set_error("device allocation failed (kNN brackets)");
    return CM_CUDA;
  }
  // first radius: the k-th neighbour distance of a surface sampled at the
  // cloud's mean xy density (ALS), later rounds grow per centre
  const DevGrid& g = ix->g;
  const double ax = g.bx1 - g.bx0, ay = g.by1 - g.by0, az = g.bz1 - g.bz0;
  const double area = ax * ay;
  double r0 = area > 0.0 ? std::sqrt((double)k / (3.141592653589793 * (double)ix->n / area))
                         : std::max(g.sx, std::max(g.sy, g.sz));
  const double rmax = std::sqrt(ax * ax + ay * ay + az * az) + std::max(g.sx, g.sy);
  static const double r0_mult = std::getenv("CMGPU_KNN_R0") ? std::atof(std::getenv("CMGPU_KNN_R0")) : 1.0;
  r0 = std::min(std::max(r0 * r0_mult, 1e-6), rmax);
  static const bool trace = std::getenv("CMGPU_KNN_TRACE") != nullptr;
  cudaEvent_t tev[16];
  int ntev = 0;
  auto mark = [&]() {
    if (trace && ntev < 16) {
      cudaEventCreate(&tev[ntev]);
      cudaEventRecord(tev[ntev++], st);
    }
  };
  mark();
  fill_f64_kernel<<<kgrid(nq), 256, 0, st>>>(rq, nq, r0); ::cmg::note_launch();
  CM_CUDA_TRY(cudaMemsetAsync(n_res, 0, 4, st));
  const uint32_t* list = perm;
  uint32_t* next = la;
  uint64_t n = nq;
  static const int kRounds = std::getenv("CMGPU_KNN_ROUNDS") ? std::atoi(std::getenv("CMGPU_KNN_ROUNDS")) : 6;
  for (int round = 0; round < kRounds && n; ++round) {
    cm_status s = radius_count_dev(ix, q, n, CM_SPHERE, r0, list, counts, nullptr, st, rq);
    if (s != CM_OK) return s;
    knn_bracket_kernel<<<kgrid(n), 256, 0, st>>>(list, (uint32_t)n, counts, k,
                                                 round == kRounds - 1, rq, f_res, f_next, rmax);
    ::cmg::note_launch();
    exclusive_scan<uint32_t, uint32_t>(f_res, n, p_res, part, 1, st);
    exclusive_scan<uint32_t, uint32_t>(f_next, n, p_next, part, 1, st);
    knn_compact_kernel<<<kgrid(n), 256, 0, st>>>(list, (uint32_t)n, f_res, p_res, f_next, p_next,
                                                 res, n_res, next, walk, n_walk);
    ::cmg::note_launch();
    add_total_kernel<<<1, 1, 0, st>>>(n_res, p_res + n); ::cmg::note_launch();
    uint32_t nn = 0;
    CM_CUDA_TRY(cudaMemcpyAsync(&nn, p_next + n, 4, cudaMemcpyDeviceToHost, st));
    CM_CUDA_TRY(cudaStreamSynchronize(st));
    mark();
    if (trace) {
      uint64_t qs[8];
      query_stats(qs, 1);
      std::fprintf(stderr, "[knn] round %d: %lu centres -> %u retry; tiles %lu fallback %lu hull %lu\n",
                   round, (unsigned long)n, nn, (unsigned long)qs[0], (unsigned long)qs[1],
                   (unsigned long)qs[2]);
    }
    list = next;
    next = next == la ? lb : la;
    n = nn;
  }
  uint32_t nres = 0;
  unsigned long long cap = 0;
  CM_CUDA_TRY(cudaMemsetAsync(cap_d, 0, 8, st));
  sum_counts_kernel<<<kgrid(nq), 256, 0, st>>>(res, n_res, counts, cap_d); ::cmg::note_launch();
  CM_CUDA_TRY(cudaMemcpyAsync(&nres, n_res, 4, cudaMemcpyDeviceToHost, st));
  CM_CUDA_TRY(cudaMemcpyAsync(&cap, cap_d, 8, cudaMemcpyDeviceToHost, st));
  CM_CUDA_TRY(cudaStreamSynchronize(st));
  if (!nres) return CM_OK;
  uint32_t* arena = nullptr;
  if (!alloc(&arena, cap + 1)) {
    set_error("device allocation failed (kNN arena)");
    return CM_CUDA;
  }
  cm_status s = radius_collect_dev(ix, q, nres, CM_SPHERE, r0, res, arena, cap + 1, toff, scnt,
                                   counts, cursor, st, nullptr, rq);
  if (s != CM_OK) return s;
  mark();
  const uint64_t need = (nres + kKWarps - 1) / kKWarps;
  const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(need, (uint64_t)sm_count() * 16));
  knn_select_kernel<<<grid, kKThreads, 0, st>>>(ix->rec, rec_of, q, res, n_res, k, arena, toff,
                                                scnt, idx, d2);
  ::cmg::note_launch();
  CM_CUDA_TRY(cudaGetLastError());
  mark();
  if (trace) {
    cudaStreamSynchronize(st);
    uint64_t qs[8];
    query_stats(qs, 1);
    std::fprintf(stderr, "[knn] resolved %u (arena %llu); collect tiles %lu fallback %lu hull %lu long %lu\n",
                 nres, cap, (unsigned long)qs[4], (unsigned long)qs[5], (unsigned long)qs[6],
                 (unsigned long)qs[7]);
    for (int i = 1; i < ntev; ++i) {
      float ms = 0;
      cudaEventElapsedTime(&ms, tev[i - 1], tev[i]);
      std::fprintf(stderr, "[knn]   phase %d: %.3f ms\n", i, ms);
    }
    for (int i = 0; i < ntev; ++i) cudaEventDestroy(tev[i]);
  }
  return CM_OK;
}

}  // namespace

cm_status knn_dev(const cm_index* ix, const double* q, uint64_t nq, uint32_t k,
                  const uint32_t* perm, uint32_t* idx, double* d2, cudaStream_t st) {
  if (nq == 0) return CM_OK;
  const Tables t = ix->tables();
  const bool glist = k > (uint32_t)kKMax;
  // chunk-local d2 scratch for large k without a d2 output (<= 1 GiB)
  const uint64_t chunk =
      glist && !d2 ? std::max<uint64_t>(1, (1ull << 27) / k) : nq;
  double* scratch = nullptr;
  if (glist && !d2) CM_CUDA_TRY(dev_alloc_t(&scratch, std::min(chunk, nq) * k, st));
  // small k: query tiles first; the centres they cannot finish are redone
  // by the shell walk over a device-built list (measured on config 3: the
  // tiles win at k = 8, 236 -> 268 M q/s; at k >= 16 the per-lane list
  // insertions and the redo share make the shell walk alone faster)
  uint32_t* redo = nullptr;
  uint32_t* n_redo = nullptr;
  const uint32_t* wperm = perm;
  // The radius-bracket path (knn_brackets) is exact but measured SLOWER on
  // config 3 (k = 8: 28-54 ms against 14.8 ms for the tiles + shell walk,
  // profiles/r02/knn_brackets.log): at a quarter of the cloud as centres a
  // 32-centre tile's hull has a median of 30 columns, so 43 % of the count
  // passes' tiles fall back to one centre per warp. Kept behind
  // CMGPU_KNN_BRACKETS for that comparison.
  static const bool brackets = std::getenv("CMGPU_KNN_BRACKETS") != nullptr;
  static const bool legacy = std::getenv("CMGPU_KNN_LEGACY") != nullptr;
  // (k = 64 measured slower per thread than one warp per centre: 109 ms
  // against 39 ms on config 3; k = 32 with the register-list second pass:
  // 19.0 ms against 20.9 ms for one warp per centre)
  static const uint32_t thread_kmax =
      std::getenv("CMGPU_KNN_THREAD_KMAX") ? (uint32_t)std::atoi(std::getenv("CMGPU_KNN_THREAD_KMAX")) : 32u;
  if (!brackets && !legacy && k <= std::min(64u, thread_kmax)) {
    // per-thread kNN: pass 1 up to shell LFIRST, pass 2 (all shells) on the
    // centres pass 1 could not finish
    static const int lfirst_env = std::getenv("CMGPU_KNN_LFIRST") ? std::atoi(std::getenv("CMGPU_KNN_LFIRST")) : 0;
    const int lfirst = lfirst_env > 0 ? lfirst_env : 1;
    // first box radius: the k-th neighbour distance of a surface sampled at
    // the cloud's mean xy density (ALS), times a margin; 0 = Chebyshev shells
    static const double r0_mult =
        std::getenv("CMGPU_KNN_R0MULT") ? std::atof(std::getenv("CMGPU_KNN_R0MULT")) : 0.0;
    double r0 = 0.0;
    {
      const DevGrid& gg = ix->g;
      const double area = (gg.bx1 - gg.bx0) * (gg.by1 - gg.by0);
      if (r0_mult > 0.0)
        r0 = area > 0.0 ? r0_mult * std::sqrt((double)k / (3.141592653589793 * (double)ix->n / area))
                        : std::max(gg.sx, std::max(gg.sy, gg.sz));
    }
    uint32_t* redo1 = nullptr;
    uint32_t* redo2 = nullptr;
    uint32_t* nr = nullptr;  // [0] pass-1 redo count, [1] pass-2 (must stay 0)
    CM_CUDA_TRY(dev_alloc_t(&redo1, nq, st));
    CM_CUDA_TRY(dev_alloc_t(&redo2, nq, st));
    CM_CUDA_TRY(dev_alloc_t(&nr, 2, st));
    CM_CUDA_TRY(cudaMemsetAsync(nr, 0, 8, st));
    auto pass = [&](auto kern, int K, const uint32_t* list, const uint32_t* nl, int lmax,
                    uint32_t* rd, uint32_t* nrd) -> cm_status {
      const size_t smem = (size_t)K * kTThreads * 12;
      if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      int per_sm = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kTThreads, smem);
      per_sm = std::max(per_sm, 1);
      const uint64_t need = (nq + kTThreads - 1) / kTThreads;
      const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(need, (uint64_t)sm_count() * per_sm));
      kern<<<grid, kTThreads, smem, st>>>(t, q, nq, k, list, nl, lmax, idx, d2, rd, nrd, r0);
      ::cmg::note_launch();
      CM_CUDA_TRY(cudaGetLastError());
      return CM_OK;
    };
    // pass 2: the centres pass 1 left (sparse neighbourhoods: several
    // shells of span lookups for a handful of candidates) go one per WARP
    // with the list in registers (config 3 k = 8 / 16: the per-thread pass 2
    // took 3.7 / 6.7 ms for 15 % of the centres); CMGPU_KNN_REDO=thread
    // keeps the per-thread walk
    static const bool redo_thread =
        std::getenv("CMGPU_KNN_REDO") && std::string(std::getenv("CMGPU_KNN_REDO")) == "thread";
    auto redo_warp = [&](auto kern) -> cm_status {
      int per_sm = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kKThreads, 0);
      per_sm = std::max(per_sm, 1);
      const uint64_t need = (nq + kKWarps - 1) / kKWarps;
      const unsigned grid =
          (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(need, (uint64_t)sm_count() * per_sm));
      // first block of pass 2 (config 3, L0 = 1 / 2 / 3: k = 8 6.11 / 5.43 /
      // 5.84 ms, k = 16 9.35 / 8.63 / 8.34 ms)
      static const int redo_l0_env =
          std::getenv("CMGPU_KNN_REDO_L0") ? std::max(1, std::atoi(std::getenv("CMGPU_KNN_REDO_L0"))) : 0;
      const int redo_l0 = redo_l0_env ? redo_l0_env : (k <= 8 ? 2 : 3);
      kern<<<grid, kKThreads, 0, st>>>(t, q, 0, nq, k, redo1, idx, d2, nr, redo_l0);
      ::cmg::note_launch();
      CM_CUDA_TRY(cudaGetLastError());
      return CM_OK;
    };
    auto both = [&](auto kern, int K) -> cm_status {
      const cm_status s1 = pass(kern, K, perm, nullptr, lfirst, redo1, nr);
      if (s1 != CM_OK) return s1;
      if (!redo_thread && k <= 32) {
        switch (ix->opts.flavor) {
          case CM_DENSE: return redo_warp(knn_warp_reg_kernel<CM_DENSE>);
          case CM_SPARSE: return redo_warp(knn_warp_reg_kernel<CM_SPARSE>);
          default: return redo_warp(knn_warp_reg_kernel<CM_MIXED>);
        }
      }
      return pass(kern, K, redo1, nr, 1 << 30, redo2, nr + 1);
    };
    auto by_k = [&](auto k8, auto k16, auto k32, auto k64) -> cm_status {
      if (k <= 8) return both(k8, 8);
      if (k <= 16) return both(k16, 16);
      if (k <= 32) return both(k32, 32);
      return both(k64, 64);
    };
    cm_status s;
    switch (ix->opts.flavor) {
      case CM_DENSE:
        s = by_k(knn_thread_kernel<CM_DENSE, 8>, knn_thread_kernel<CM_DENSE, 16>,
                 knn_thread_kernel<CM_DENSE, 32>, knn_thread_kernel<CM_DENSE, 64>);
        break;
      case CM_SPARSE:
        s = by_k(knn_thread_kernel<CM_SPARSE, 8>, knn_thread_kernel<CM_SPARSE, 16>,
                 knn_thread_kernel<CM_SPARSE, 32>, knn_thread_kernel<CM_SPARSE, 64>);
        break;
      default:
        s = by_k(knn_thread_kernel<CM_MIXED, 8>, knn_thread_kernel<CM_MIXED, 16>,
                 knn_thread_kernel<CM_MIXED, 32>, knn_thread_kernel<CM_MIXED, 64>);
    }
    dev_free(redo1, st);
    dev_free(redo2, st);
    dev_free(nr, st);
    if (scratch) dev_free(scratch, st);
    return s;
  }
  if (!glist && !ix->global_ids && brackets) {
    // radius brackets first; the shell walk takes what they leave
    CM_CUDA_TRY(dev_alloc_t(&redo, nq, st));
    CM_CUDA_TRY(dev_alloc_t(&n_redo, 1, st));
    CM_CUDA_TRY(cudaMemsetAsync(n_redo, 0, 4, st));
    const cm_status bs = knn_brackets(ix, q, nq, k, perm, idx, d2, st, redo, n_redo);
    if (bs != CM_OK) {
      dev_free(redo, st);
      dev_free(n_redo, st);
      return bs;
    }
    wperm = redo;
  } else if (!glist && k <= kKnnTileMax) {
    CM_CUDA_TRY(dev_alloc_t(&redo, nq, st));
    CM_CUDA_TRY(dev_alloc_t(&n_redo, 1, st));
    CM_CUDA_TRY(cudaMemsetAsync(n_redo, 0, 4, st));
    auto tiles = [&](auto kern, size_t smem) -> cm_status {
      if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      int per_sm = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kKThreads, smem);
      per_sm = std::max(per_sm, 1);
      const uint64_t need = ((nq + 31) / 32 + kKWarps - 1) / kKWarps;
      const unsigned grid =
          (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(need, (uint64_t)sm_count() * per_sm));
      kern<<<grid, kKThreads, smem, st>>>(t, q, nq, k, perm, idx, d2, redo, n_redo); ::cmg::note_launch();
      CM_CUDA_TRY(cudaGetLastError());
      return CM_OK;
    };
    const size_t s8 = kKWarps * sizeof(KnnTileSmem<8>);
    cm_status ts;
#if CM_KNN_TILE_MAX > 8
    const size_t s16 = kKWarps * sizeof(KnnTileSmem<16>);
    if (k > 8) {
      switch (ix->opts.flavor) {
        case CM_DENSE:
          ts = tiles(knn_tile_kernel<CM_DENSE, 16>, s16);
          break;
        case CM_SPARSE:
          ts = tiles(knn_tile_kernel<CM_SPARSE, 16>, s16);
          break;
        default:
          ts = tiles(knn_tile_kernel<CM_MIXED, 16>, s16);
      }
    } else
#endif
    switch (ix->opts.flavor) {
      case CM_DENSE:
        ts = tiles(knn_tile_kernel<CM_DENSE, 8>, s8);
        break;
      case CM_SPARSE:
        ts = tiles(knn_tile_kernel<CM_SPARSE, 8>, s8);
        break;
      default:
        ts = tiles(knn_tile_kernel<CM_MIXED, 8>, s8);
    }
    if (ts != CM_OK) {
      dev_free(redo, st);
      dev_free(n_redo, st);
      return ts;
    }
    wperm = redo;
  }
  // 16 < k <= 64: histogram selection first; what it leaves goes to the
  // register-list walk (k <= 32, from block 3) or the shell walk
  // (config 3: k = 64 38.8 / 35.7 ms with 2 / 6 levels against 39.3 ms for
  // the shell walk alone; k = 32 20.3 ms, where the per-thread first pass
  // plus the register-list second pass takes 19.0 ms and is the default)
  static const int hist_lmax =
      std::getenv("CMGPU_KNN_HIST") ? std::atoi(std::getenv("CMGPU_KNN_HIST")) : 6;
  int reg_l0 = 1;
  if (hist_lmax > 0 && !legacy && !brackets && !glist && !redo && k > 16 && k <= 64) {
    CM_CUDA_TRY(dev_alloc_t(&redo, nq, st));
    CM_CUDA_TRY(dev_alloc_t(&n_redo, 1, st));
    CM_CUDA_TRY(cudaMemsetAsync(n_redo, 0, 4, st));
    auto runh = [&](auto kern) -> cm_status {
      int per_sm = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kKThreads, 0);
      per_sm = std::max(per_sm, 1);
      const uint64_t need = (nq + kKWarps - 1) / kKWarps;
      const unsigned grid =
          (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(need, (uint64_t)sm_count() * per_sm));
      kern<<<grid, kKThreads, 0, st>>>(t, q, nq, k, perm, idx, d2, redo, n_redo, hist_lmax);
      ::cmg::note_launch();
      CM_CUDA_TRY(cudaGetLastError());
      return CM_OK;
    };
    cm_status hs;
    switch (ix->opts.flavor) {
      case CM_DENSE: hs = runh(knn_hist_kernel<CM_DENSE>); break;
      case CM_SPARSE: hs = runh(knn_hist_kernel<CM_SPARSE>); break;
      default: hs = runh(knn_hist_kernel<CM_MIXED>);
    }
    if (hs != CM_OK) {
      dev_free(redo, st);
      dev_free(n_redo, st);
      return hs;
    }
    wperm = redo;
    reg_l0 = hist_lmax >= 2 ? 3 : 1;
  }
  // 16 < k <= 32: one warp per centre with the list in registers
  static const bool reg32 = !(std::getenv("CMGPU_KNN_REG32") && std::atoi(std::getenv("CMGPU_KNN_REG32")) == 0);
  if (reg32 && !legacy && !glist && k <= 32) {
    auto runr = [&](auto kern) -> cm_status {
      int per_sm = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kKThreads, 0);
      per_sm = std::max(per_sm, 1);
      const uint64_t need = (nq + kKWarps - 1) / kKWarps;
      const unsigned grid =
          (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(need, (uint64_t)sm_count() * per_sm));
      kern<<<grid, kKThreads, 0, st>>>(t, q, 0, nq, k, wperm, idx, d2, n_redo, reg_l0);
      ::cmg::note_launch();
      CM_CUDA_TRY(cudaGetLastError());
      return CM_OK;
    };
    cm_status s;
    switch (ix->opts.flavor) {
      case CM_DENSE: s = runr(knn_warp_reg_kernel<CM_DENSE>); break;
      case CM_SPARSE: s = runr(knn_warp_reg_kernel<CM_SPARSE>); break;
      default: s = runr(knn_warp_reg_kernel<CM_MIXED>);
    }
    if (redo) dev_free(redo, st);
    if (n_redo) dev_free(n_redo, st);
    return s;
  }
  auto run = [&](auto kern) -> cm_status {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kKThreads, 0);
    per_sm = std::max(per_sm, 1);
    for (uint64_t s0 = 0; s0 < nq; s0 += chunk) {
      const uint64_t s1 = std::min(nq, s0 + chunk);
      const uint64_t need = (s1 - s0 + kKWarps - 1) / kKWarps;
      const unsigned grid =
          (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(need, (uint64_t)sm_count() * per_sm));
      kern<<<grid, kKThreads, 0, st>>>(t, q, s0, s1, k, wperm, idx, d2, scratch, n_redo); ::cmg::note_launch();
      CM_CUDA_TRY(cudaGetLastError());
    }
    return CM_OK;
  };
  cm_status s;
  switch (ix->opts.flavor) {
    case CM_DENSE:
      s = glist ? run(knn_warp_kernel<CM_DENSE, true>) : run(knn_warp_kernel<CM_DENSE, false>);
      break;
    case CM_SPARSE:
      s = glist ? run(knn_warp_kernel<CM_SPARSE, true>) : run(knn_warp_kernel<CM_SPARSE, false>);
      break;
    default:
      s = glist ? run(knn_warp_kernel<CM_MIXED, true>) : run(knn_warp_kernel<CM_MIXED, false>);
  }
  if (scratch) dev_free(scratch, st);
  if (redo) dev_free(redo, st);
  if (n_redo) dev_free(n_redo, st);
  return s;
}

}  // namespace cmg
