// Batched fixed-radius queries (sphere / cube) on sm_100a.
// Replaces kernel_search<Kernel> (search.hpp:102-127) for a batch of centres.
//
// Candidate enumeration is exactly the reference's: every point of every
// voxel of clamped_range(c +- r) (grid.cpp:90-114). The points of one
// (i, j) column inside [k0, k1] are one contiguous span of the cell-sorted
// records (global_index is k-fastest, grid.hpp:65-67), so a query is a
// handful of spans.
//
// Work decomposition:
//  * queries are radix-sorted by cell key, so a warp's 32 consecutive
//    queries are spatial neighbours (a query TILE);
//  * a tile whose clamped ranges have a compact hull (<= 32 columns) walks
//    the hull's points once, warp-uniformly (one L1 broadcast per record);
//    each lane tests every point against its own query, keeping only points
//    whose voxel is in that query's own range, with the reference's exact
//    predicate arithmetic;
//  * hits go to a per-lane row buffer in shared memory; each row is then
//    sorted by the whole warp (register bitonic) and written coalesced;
//  * lanes whose rows overflow the buffer, and tiles that are not compact,
//    are answered one query per warp (flattened spans, 32 candidates/step).
//
// Passes: COUNT (counts + QueryStats::points_tested), DIGEST (count + set
// digest), FILL (sorted rows at caller row_ptr), COLLECT (single pass: sorted
// rows into a scratch arena at atomically allocated offsets; a gather copies
// them into CSR order after the row_ptr scan).
#include <algorithm>
#include <type_traits>
#include <cstdlib>

#include "index.cuh"
#include "sort_scan.cuh"
#include "tile_walk.cuh"

namespace cmg {

namespace {

using namespace ::cmg::tw;  // tile_walk.cuh

#ifndef CM_FILL_MINB
// blocks per SM the FILL walk is compiled for: 4 gives it 128 registers and
// no spills (wide FILL at r = 2.5: 41 -> 34 ms per launch; 5 spilled)
#define CM_FILL_MINB 4
#endif
#ifndef CM_CUBE_MINB
#define CM_CUBE_MINB CM_QTILE_MINB  // blocks per SM for the cube kernel's other passes
#endif
#ifndef CM_CUBE_GROUP
#define CM_CUBE_GROUP 4
#endif
constexpr int kQThreads = 128;
constexpr int kQWarps = kQThreads / 32;
#ifndef CM_LANE_ROW_CAP
#define CM_LANE_ROW_CAP 128
#endif
#ifndef CM_QTILE_MINB
#define CM_QTILE_MINB 5
#endif
constexpr int kLaneRowCap = CM_LANE_ROW_CAP;          // per-lane row buffer
// the FILL row translation and the gather's warp sort of 97..cap rows hold a
// row in 4 registers per lane (4 x 32 = 128 handles)
static_assert(kLaneRowCap >= 97 && kLaneRowCap <= 128, "CM_LANE_ROW_CAP must be in [97, 128]");
// Per warp: the tile path's per-lane rows (u16 hit keys, interleaved with
// stride 33) followed by the cp.async staging double buffer; the one-query
// path reuses the whole region as a u32 buffer.
constexpr int kRowKeyBytes = kLaneRowCap * 33 * 2;
constexpr int kStageBytes = 64 * 32;
constexpr int kRowWarpBytes = kRowKeyBytes + kStageBytes;
// FILL launches: the row area holds the wide tile's per-lane HANDLE buffers
// (u32, kFillCap per lane, stride 33) — flushes then need no record lookups —
// and still fits the compact tile's u16 key rows.
constexpr int kFillCap = 64;
// + one scratch slot per lane: the walk stores every record's handle at the
// lane's next slot unconditionally (no branch per hit) and advances on hits
constexpr int kFillRowBytes = ((kFillCap + 1) * 33 * 4 + 15) / 16 * 16 > kRowKeyBytes
                                  ? ((kFillCap + 1) * 33 * 4 + 15) / 16 * 16
                                  : kRowKeyBytes;
template <int MODE>
__host__ __device__ constexpr int row_area_bytes() {
  return MODE == 1 /* MODE_FILL */ ? kFillRowBytes : kRowKeyBytes;
}
template <int MODE>
__host__ __device__ constexpr int warp_smem_bytes() { return row_area_bytes<MODE>() + kStageBytes; }
#ifndef CM_TILE_SPLIT
#define CM_TILE_SPLIT 1  // COLLECT: sparse tiles answered in parts (halves, quarters, ...)
#endif
#ifndef CM_TILE_SPLIT_MIN
#define CM_TILE_SPLIT_MIN 4  // parts are not halved below this many lanes
#endif
constexpr int kWideMaxCols = 4096;                    // wide tiles: hull column limit
constexpr int kRowCap = kRowWarpBytes / 4;            // one-query row buffer (u32)
constexpr int kSortCap = (kRowCap - 512) / 2;         // one-query row sorted in smem
constexpr int kBigSmemCap = 32768;                    // block sort in smem (128 KB)

enum { MODE_COUNT = 0, MODE_FILL = 1, MODE_DIGEST = 2, MODE_COLLECT = 3 };

// Tile statistics (cm_debug_query_stats): count pass [0..3], row passes
// (fill / collect) [4..7]: tiles, non-compact tiles, hull points, and
// in-range candidates (count) / long rows answered per query (row passes).
__device__ unsigned long long g_qstats[8];
// Tile counters (cm_debug_query_stats): compiled into the CHECKED library
// only. They accumulate per warp in shared memory (one writer, lane 0) and
// reach g_qstats once per warp at the end of the kernel — but the single-lane
// updates alone, inside the tile loop, cost the wide-tile passes half their
// speed (the warp stays on its divergent path for the shuffles and votes
// that follow; global atomics or shared memory made no difference). Without
// them: config 2 digests 11.2 / 6.7 / 2.4 -> 22.9 / 12.4 / 4.3 M q/s, the count
// pass at r = 5 14.4 -> 10.5 ms, the count pass over every 7th / 50th point
// of config 1 6.75 / 2.77 -> 3.0 / 0.9 ms; the compact COLLECT walk is
// unchanged (9.88 -> 9.86 ms).
#ifndef CM_QSTATS
#ifdef CMGPU_CHECKED
#define CM_QSTATS 1
#else
#define CM_QSTATS 0
#endif
#endif
#define QSTAT_ADD(i, v) do { if (CM_QSTATS) wqs[i] += (unsigned long long)(v); } while (0)

// Kernel outputs; which fields are used depends on the pass.
struct Out {
  uint32_t* counts;
  uint64_t* tested;
  uint64_t* digests;
  const uint64_t* row_ptr;        // FILL
  uint32_t* cols;                 // FILL
  uint32_t* temp;                 // COLLECT arena
  uint64_t cap;                   // COLLECT arena capacity (entries)
  uint64_t* toff;                 // COLLECT arena offset, by query
  uint32_t* scnt;                 // COLLECT row length, by query
  unsigned long long* cursor;     // COLLECT arena bump pointer (rows padded to 4 handles)
  unsigned long long* nnz;        // COLLECT: exact handle count (or null)
  uint64_t* big_off;              // rows sorted afterwards: offset into `rows`
  uint32_t* big_len;
  uint32_t* big_q;                // COLLECT with a merge list: the row's query (or null)
  uint32_t* n_big;
  int wide_fill;                  // FILL: wide tiles may leave rows unsorted (sorted afterwards)
  uint32_t cur_q;                 // (set per call of single_query for big-row registration)
  const double* rq;               // per-centre radius by query index (kNN brackets), or null
  const double* qbox;             // per-centre kernel box {min, max} by query index, or null
  int no_wide;                    // diagnostics (CMGPU_NO_WIDE): wide tiles off
};

// Query order keys. RANGE = false: the centre's cell key, so a tile's 32
// consecutive centres are spatial neighbours. RANGE = true (radii of at most
// half a cell, where every clamped range spans 1 or 2 cells per axis): the
// key of the range's low corner voxel, times 8, plus one bit per axis for a
// 2-cell extent — centres with the same candidate voxels sort together, so
// a tile's hull is the union of few distinct ranges (dense voxels holding
// many centres, as near a TLS scanner, otherwise give every tile the whole
// 3 x 3 x 3 neighbourhood).
template <typename K, bool RANGE>
__global__ void query_keys_kernel(const double* __restrict__ q, uint64_t nq, DevGrid g,
                                  K* __restrict__ keys, uint32_t* __restrict__ vals, double r,
                                  int kind) {
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < nq;
       p += (uint64_t)gridDim.x * blockDim.x) {
    const double cx = q[3 * p], cy = q[3 * p + 1], cz = q[3 * p + 2];
    uint64_t i = axis_index(cx, g.ox, g.sx, g.nx);
    uint64_t j = axis_index(cy, g.oy, g.sy, g.ny);
    uint64_t k = g.mode3d ? axis_index(cz, g.oz, g.sz, g.nz) : 0;
    uint64_t ext = 0;
    if (RANGE) {
      Range R;
      if (clamped_range(g, cx, cy, cz, r, &R, kind)) {
        i = R.i0, j = R.j0, k = R.k0;
        ext = ((uint64_t)(R.i1 > R.i0) << 2) | ((uint64_t)(R.j1 > R.j0) << 1) |
              (uint64_t)(R.k1 > R.k0);
      }
    }
    const uint64_t cell = i * (g.ny * g.nz) + j * g.nz + k;
    keys[p] = (K)(RANGE ? cell * 8 + ext : cell);
    vals[p] = (uint32_t)p;
  }
}

// 2D Morton order of the centre's (i, j) column, voxel k in the low bits:
// for SPARSE centre sets (a random quarter of the cloud, as kNN config 3)
// 32 consecutive centres then form a compact patch of columns instead of a
// strip along j, so a tile's hull stays within the compact-tile limit.
__device__ __forceinline__ uint64_t interleave2(uint64_t a, uint64_t b) {
  // a on even bits, b on odd bits
  uint64_t x = 0;
#pragma unroll
  for (int i = 0; i < 21; ++i) x |= (((a >> i) & 1ull) << (2 * i)) | (((b >> i) & 1ull) << (2 * i + 1));
  return x;
}
template <typename K>
__global__ void query_morton_kernel(const double* __restrict__ q, uint64_t nq, DevGrid g,
                                    K* __restrict__ keys, uint32_t* __restrict__ vals, int bz) {
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < nq;
       p += (uint64_t)gridDim.x * blockDim.x) {
    const double cx = q[3 * p], cy = q[3 * p + 1], cz = q[3 * p + 2];
    const uint64_t i = axis_index(cx, g.ox, g.sx, g.nx);
    const uint64_t j = axis_index(cy, g.oy, g.sy, g.ny);
    const uint64_t k = g.mode3d ? axis_index(cz, g.oz, g.sz, g.nz) : 0;
    keys[p] = (K)((interleave2(j, i) << bz) | k);
    vals[p] = (uint32_t)p;
  }
}

// Flip-variant bitonic sort (ascending) of a[0..n) by `nthreads` cooperating
// threads (tid in [0, nthreads)). Indices >= n behave as +inf, so n need not
// be a power of two. `sync` orders the stages.
template <class Sync>
__device__ __forceinline__ void bitonic_sort(uint32_t* a, uint32_t n, uint32_t tid,
                                             uint32_t nthreads, Sync sync) {
  uint32_t P = 1;
  while (P < n) P <<= 1;
  for (uint32_t k = 2; k <= P; k <<= 1) {
    for (uint32_t i = tid; i < P; i += nthreads) {
      const uint32_t p = i ^ (k - 1);
      if (p > i && p < n) {
        const uint32_t x = a[i], y = a[p];
        if (x > y) {
          a[i] = y;
          a[p] = x;
        }
      }
    }
    sync();
    for (uint32_t j = k >> 2; j > 0; j >>= 1) {
      for (uint32_t i = tid; i < P; i += nthreads) {
        const uint32_t p = i ^ j;
        if (p > i && p < n) {
          const uint32_t x = a[i], y = a[p];
          if (x > y) {
            a[i] = y;
            a[p] = x;
          }
        }
      }
      sync();
    }
  }
}

// 32-wide register bitonic sort, one value per lane, ascending by lane.
__device__ __forceinline__ uint32_t warp_sort32(uint32_t v, int lane) {
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const uint32_t o = __shfl_xor_sync(0xffffffffu, v, j);
      const bool up = (lane & k) == 0 || k == 32;
      const bool lower = (lane & j) == 0;
      v = (lower == up) ? min(v, o) : max(v, o);
    }
  }
  return v;
}

// One query answered by a whole warp (the fallback when a 32-query tile is
// not compact): ncol column spans flattened, 32 candidates per step.
// Ascending bitonic sort of P = 32 * ITEMS u32 keys held by one warp in
// registers, striped: element e = r * 32 + lane lives in v[r] of `lane`.
// Exchanges at distance < 32 go through shuffles, the rest stay in-lane.
template <int ITEMS>
__device__ __forceinline__ void warp_sort_regs(uint32_t (&v)[ITEMS], int lane) {
  constexpr int LOGP = ITEMS == 1    ? 5
                       : ITEMS == 2  ? 6
                       : ITEMS == 4  ? 7
                       : ITEMS == 8  ? 8
                       : ITEMS == 16 ? 9
                                     : 10;
#pragma unroll
  for (int lk = 1; lk <= LOGP; ++lk) {
    const int k = 1 << lk;
#pragma unroll
    for (int lj = lk - 1; lj >= 0; --lj) {
      const int j = 1 << lj;
      if (lj < 5) {
#pragma unroll
        for (int r = 0; r < ITEMS; ++r) {
          const int e = r * 32 + lane;
          const uint32_t o = __shfl_xor_sync(0xffffffffu, v[r], j);
          const bool asc = (e & k) == 0;
          const bool lower = (lane & j) == 0;
          v[r] = (lower == asc) ? min(v[r], o) : max(v[r], o);
        }
      } else {
        const int jr = j >> 5;
#pragma unroll
        for (int r = 0; r < ITEMS; ++r) {
          if ((r & jr) == 0) {
            const int e = r * 32 + lane;
            const bool asc = (e & k) == 0;
            const uint32_t x = v[r], y = v[r | jr];
            v[r] = asc ? min(x, y) : max(x, y);
            v[r | jr] = asc ? max(x, y) : min(x, y);
          }
        }
      }
    }
  }
}

// Ascending sorting network over P registers of ONE thread (compile-time
// indices only, so v stays in registers): Batcher's odd-even merge sort
// (543 compare-exchanges at P = 64 against the bitonic network's 672; fewer
// instructions and a smaller unrolled body). CM_LANE_BITONIC selects the
// bitonic network below instead.
template <int P>
__device__ __forceinline__ void lane_ce(uint32_t (&v)[P], int i, int j) {
  const uint32_t a = v[i], b = v[j];
  v[i] = min(a, b);
  v[j] = max(a, b);
}
// odd-even merge of v[LO, LO + N) whose halves are sorted, stride R
template <int P, int LO, int N, int R>
struct OemMerge {
  __device__ __forceinline__ static void run(uint32_t (&v)[P]) {
    if constexpr (2 * R < N) {
      OemMerge<P, LO, N, 2 * R>::run(v);
      OemMerge<P, LO + R, N, 2 * R>::run(v);
#pragma unroll
      for (int i = LO + R; i + R < LO + N; i += 2 * R) lane_ce<P>(v, i, i + R);
    } else {
      lane_ce<P>(v, LO, LO + R);
    }
  }
};
template <int P, int LO, int N>
struct OemSort {
  __device__ __forceinline__ static void run(uint32_t (&v)[P]) {
    if constexpr (N > 1) {
      OemSort<P, LO, N / 2>::run(v);
      OemSort<P, LO + N / 2, N / 2>::run(v);
      OemMerge<P, LO, N, 1>::run(v);
    }
  }
};
template <int P>
__device__ __forceinline__ void lane_sort_oem(uint32_t (&v)[P]) {
  OemSort<P, 0, P>::run(v);
}

template <int P>
__device__ __forceinline__ void lane_sort_bitonic(uint32_t (&v)[P]) {
#pragma unroll
  for (int k = 2; k <= P; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
#pragma unroll
      for (int i = 0; i < P; ++i) {
        const int p = i ^ j;
        if (p > i) {
          const uint32_t a = v[i], b = v[p];
          if ((i & k) == 0) {
            v[i] = min(a, b);
            v[p] = max(a, b);
          } else {
            v[i] = max(a, b);
            v[p] = min(a, b);
          }
        }
      }
    }
  }
}

template <int P>
__device__ __forceinline__ void lane_sort_regs(uint32_t (&v)[P]) {
#ifdef CM_LANE_BITONIC
  lane_sort_bitonic<P>(v);
#else
  lane_sort_oem<P>(v);
#endif
}

// Each lane sorts its own interleaved row srow[i * 33 + lane], i < len
// (len <= P), in registers.
template <int P>
__device__ __forceinline__ void lane_sort_row(uint32_t* srow, int lane, uint32_t len) {
  uint32_t v[P];
#pragma unroll
  for (int i = 0; i < P; ++i) v[i] = (uint32_t)i < len ? srow[i * 33 + lane] : 0xffffffffu;
  lane_sort_regs<P>(v);
#pragma unroll
  for (int i = 0; i < P; ++i)
    if ((uint32_t)i < len) srow[i * 33 + lane] = v[i];
}

// Sorts lane l's interleaved row (srow[i * 33 + l], i < len) with the whole
// warp and writes it ascending to dst[0..len) (coalesced).
template <int ITEMS>
__device__ __forceinline__ void warp_sort_row_out(const uint32_t* srow, int l, uint32_t len,
                                                  uint32_t* dst, int lane) {
  uint32_t v[ITEMS];
#pragma unroll
  for (int r = 0; r < ITEMS; ++r) {
    const uint32_t e = r * 32 + lane;
    v[r] = e < len ? srow[e * 33 + l] : 0xffffffffu;
  }
  warp_sort_regs<ITEMS>(v, lane);
#pragma unroll
  for (int r = 0; r < ITEMS; ++r) {
    const uint32_t e = r * 32 + lane;
    if (e < len) dst[e] = v[r];
  }
}

// A read-only global load the compiler cannot merge with an earlier one (so
// values can be re-read instead of kept live in registers).
__device__ __forceinline__ double ldg_opaque(const double* p) {
  double v;
  asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

// Predicated 16-bit shared store (no branch around it).
__device__ __forceinline__ void sts_u16_if(uint32_t addr, uint32_t v, bool p) {
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n @q st.shared.u16 [%0], %1;\n}\n" ::"r"(addr),
      "h"((unsigned short)v), "r"((uint32_t)p));
}

template <int CUBE>
__device__ __forceinline__ bool pred(const Predicate& P, double x, double y, double z) {
  if (CUBE == 1)  // closed box (geometry.hpp:48-51)
    return (x >= P.lx) & (x <= P.hx) & (y >= P.ly) & (y <= P.hy) & (z >= P.lz) & (z <= P.hz);
  if (CUBE == 2) {  // vertical cylinder (geometry.hpp:107-110)
    const double dx = __dsub_rn(x, P.cx), dy = __dsub_rn(y, P.cy);
    return (z >= P.lz) & (z <= P.hz) & (__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)) <= P.rr);
  }
  return sqdist(x, y, z, P.cx, P.cy, P.cz) <= P.rr;  // sphere (geometry.hpp:82-84)
}



// One query answered by a whole warp: count pass over the flattened spans.
template <int FLAVOR, int CUBE, bool DIG>
__device__ __forceinline__ void warp_query_count(const Tables& t, double cx, double cy, double cz,
                                                 double r, int lane, uint32_t* cnt_out,
                                                 uint64_t* tested_out, uint64_t* dig_out,
                                                 const double* box) {
  Range R;
  const bool ok = clamped_range_warp(t.g, cx, cy, cz, r, lane, &R, CUBE, box);
  Predicate P;
  P.init(cx, cy, cz, r, CUBE, box);
  uint32_t cnt = 0;
  uint64_t ntested = 0, dig = 0;
  if (ok) {
    const uint64_t nj = R.j1 - R.j0 + 1;
    const uint64_t ncol = (R.i1 - R.i0 + 1) * nj;
    for (uint64_t cb = 0; cb < ncol; cb += 32) {
      const uint64_t c = cb + lane;
      uint32_t b = 0, e = 0;
      if (c < ncol) column_span<FLAVOR>(t, R.i0 + c / nj, R.j0 + c % nj, R.k0, R.k1, &b, &e);
      const uint32_t len = e - b;
      const uint32_t incl = warp_incl_scan(len);
      const uint32_t excl = incl - len;
      const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
      ntested += total;
      for (uint32_t t0 = 0; t0 < total; t0 += 32) {
        const uint32_t tt = t0 + lane;
        int L = 0;
#pragma unroll
        for (int sft = 16; sft > 0; sft >>= 1) {
          const uint32_t v = __shfl_sync(0xffffffffu, incl, L + sft - 1);
          if (v <= tt) L += sft;
        }
        const uint32_t bL = __shfl_sync(0xffffffffu, b, L);
        const uint32_t xL = __shfl_sync(0xffffffffu, excl, L);
        bool hit = false;
        if (tt < total) {
          const PointRec pr = load_rec(t.rec + bL + (tt - xL));
          hit = pred<CUBE>(P, pr.x, pr.y, pr.z);
          if (DIG && hit) dig += mix64(pr.id);
        }
        cnt += __popc(__ballot_sync(0xffffffffu, hit));
      }
    }
  }
  if (DIG) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dig += __shfl_xor_sync(0xffffffffu, dig, o);
  }
  *cnt_out = cnt;
  *tested_out = ntested;
  *dig_out = dig;
}

// Warp LSD radix sort of a[0..n) (u32, keys < 2^bits) with 9-bit digits,
// ping-ponging through tmp; `cnt` holds 512 counters. Stable per pass
// (ranks inside a 32-element chunk from per-bit ballots). Returns the buffer
// holding the result.
__device__ __noinline__ uint32_t* warp_radix_sort(uint32_t* a, uint32_t* tmp, uint32_t* cnt,
                                                  uint32_t n, int bits, int lane, uint32_t lt) {
  constexpr int R = 9;
  constexpr uint32_t M = (1u << R) - 1;
  for (int sh = 0; sh < bits; sh += R) {
    for (int d = lane; d <= (int)M; d += 32) cnt[d] = 0;
    __syncwarp();
    for (uint32_t i = lane; i < n; i += 32) atomicAdd(&cnt[(a[i] >> sh) & M], 1u);
    __syncwarp();
    // exclusive scan of the 512 counters: 16 per lane
    uint32_t loc[16], sum = 0;
#pragma unroll
    for (int x = 0; x < 16; ++x) {
      loc[x] = cnt[lane * 16 + x];
      sum += loc[x];
    }
    const uint32_t inc = warp_incl_scan(sum);
    uint32_t run = inc - sum;
#pragma unroll
    for (int x = 0; x < 16; ++x) {
      cnt[lane * 16 + x] = run;
      run += loc[x];
    }
    __syncwarp();
    for (uint32_t base = 0; base < n; base += 32) {
      const uint32_t i = base + lane;
      const bool valid = i < n;
      const uint32_t v = valid ? a[i] : 0u;
      const uint32_t d = valid ? ((v >> sh) & M) : (M + 1);
      // peer group: one ballot per digit bit (faster than __match_any_sync,
      // as in the build's radix downsweep)
      uint32_t peers = __ballot_sync(0xffffffffu, valid);
#pragma unroll
      for (int bb = 0; bb < R; ++bb) {
        const bool bit = (d >> bb) & 1u;
        const uint32_t m = __ballot_sync(0xffffffffu, bit);
        peers &= bit ? m : ~m;
      }
      uint32_t pos = 0;
      if (valid) pos = cnt[d] + __popc(peers & lt);
      __syncwarp();
      if (valid) {
        tmp[pos] = v;
        if ((peers & lt) == 0) cnt[d] = pos + __popc(peers);
      }
      __syncwarp();
    }
    uint32_t* t2 = a;
    a = tmp;
    tmp = t2;
  }
  return a;
}

// Sorts buf[0..n) (n <= kSortCap) ascending with the cheapest method for n;
// returns where the result is (buf, or the scratch half for radix).
__device__ __forceinline__ const uint32_t* warp_sort_buffer(uint32_t* buf, uint32_t n, int bits,
                                                            int lane, uint32_t lt) {
  if (n <= 1) return buf;
  if (n <= 32) {
    uint32_t v = lane < (int)n ? buf[lane] : 0xffffffffu;
    v = warp_sort32(v, lane);
    __syncwarp();
    if (lane < (int)n) buf[lane] = v;
    __syncwarp();
    return buf;
  }
  if (n <= 128) {
    uint32_t v[4];
#pragma unroll
    for (int r2 = 0; r2 < 4; ++r2) {
      const uint32_t e = r2 * 32 + lane;
      v[r2] = e < n ? buf[e] : 0xffffffffu;
    }
    warp_sort_regs<4>(v, lane);
    __syncwarp();
#pragma unroll
    for (int r2 = 0; r2 < 4; ++r2) {
      const uint32_t e = r2 * 32 + lane;
      if (e < n) buf[e] = v[r2];
    }
    __syncwarp();
    return buf;
  }
  return warp_radix_sort(buf, buf + kSortCap, buf + 2 * kSortCap, n, bits, lane, lt);
}

// One query answered by a whole warp: walks its flattened spans (32
// candidates per step). Hits go to buf[0..cap) (then `direct` must be null),
// or straight to `direct` in visit order. Returns the hit count.
template <int FLAVOR, int CUBE>
__device__ __forceinline__ uint32_t warp_query_walk(const Tables& t, double cx, double cy,
                                                    double cz, double r, int lane, uint32_t lt,
                                                    uint32_t* buf, uint32_t cap,
                                                    uint32_t* direct, const double* box) {
  Range R;
  const bool ok = clamped_range_warp(t.g, cx, cy, cz, r, lane, &R, CUBE, box);
  Predicate P;
  P.init(cx, cy, cz, r, CUBE, box);
  uint32_t cnt = 0;
  if (ok) {
    const uint64_t nj = R.j1 - R.j0 + 1;
    const uint64_t ncol = (R.i1 - R.i0 + 1) * nj;
    for (uint64_t cb = 0; cb < ncol; cb += 32) {
      const uint64_t c = cb + lane;
      uint32_t b = 0, e = 0;
      if (c < ncol) column_span<FLAVOR>(t, R.i0 + c / nj, R.j0 + c % nj, R.k0, R.k1, &b, &e);
      const uint32_t ln = e - b;
      const uint32_t incl = warp_incl_scan(ln);
      const uint32_t excl = incl - ln;
      const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
      for (uint32_t t0 = 0; t0 < total; t0 += 32) {
        const uint32_t tt = t0 + lane;
        int L = 0;
#pragma unroll
        for (int sft = 16; sft > 0; sft >>= 1) {
          const uint32_t v = __shfl_sync(0xffffffffu, incl, L + sft - 1);
          if (v <= tt) L += sft;
        }
        const uint32_t bL = __shfl_sync(0xffffffffu, b, L);
        const uint32_t xL = __shfl_sync(0xffffffffu, excl, L);
        bool hit = false;
        uint32_t id = 0;
        if (tt < total) {
          const PointRec pr = load_rec(t.rec + bL + (tt - xL));
          hit = pred<CUBE>(P, pr.x, pr.y, pr.z);
          id = pr.id;
        }
        const uint32_t m = __ballot_sync(0xffffffffu, hit);
        if (hit) {
          const uint32_t off = cnt + __popc(m & lt);
          if (direct) direct[off] = id;
          else if (off < cap) buf[off] = id;
        }
        cnt += __popc(m);
      }
    }
  }
  __syncwarp();
  return cnt;
}

// Writes the buffered, sorted row, or (rows > kSortCap) walks again straight
// into dst and registers the row for the block sort.
template <int FLAVOR, int CUBE>
__device__ __forceinline__ void warp_row_out(const Tables& t, double cx, double cy, double cz,
                                             double r, int lane, uint32_t lt, uint32_t* wbuf,
                                             uint32_t cnt, uint32_t* dst, uint64_t big_base,
                                             const Out& o, const double* box) {
  if (cnt <= (uint32_t)kSortCap) {
    const int bits = 32 - __clz((int)max(1u, (uint32_t)(t.n - 1)));
    const uint32_t* res = warp_sort_buffer(wbuf, cnt, bits, lane, lt);
    for (uint32_t x = lane; x < cnt; x += 32) dst[x] = res[x];
  } else {
    warp_query_walk<FLAVOR, CUBE>(t, cx, cy, cz, r, lane, lt, nullptr, 0, dst, box);
    if (lane == 0) {
      const uint32_t slot = atomicAdd(o.n_big, 1u);
      o.big_off[slot] = big_base;
      o.big_len[slot] = cnt;
      if (o.big_q) o.big_q[slot] = o.cur_q;
    }
  }
  __syncwarp();
}

// One query, one warp, any pass.
template <int FLAVOR, int MODE, int CUBE>
__device__ __forceinline__ void single_query(const Tables& t, uint32_t qi, uint64_t spos,
                                             double cx, double cy, double cz, double r, int lane,
                                             uint32_t lt, const Out& o, uint32_t* wbuf) {
  const double* box = o.qbox ? o.qbox + 6 * (uint64_t)qi : nullptr;
  if (MODE == MODE_COUNT || MODE == MODE_DIGEST) {
    uint32_t cnt;
    uint64_t tested, dig;
    warp_query_count<FLAVOR, CUBE, MODE == MODE_DIGEST>(t, cx, cy, cz, r, lane, &cnt, &tested,
                                                        &dig, box);
    if (lane == 0) {
      if (o.counts) o.counts[qi] = cnt;
      if (MODE == MODE_COUNT && o.tested) o.tested[qi] = tested;
      if (MODE == MODE_DIGEST) o.digests[qi] = dig;
    }
  } else if (MODE == MODE_FILL) {
    const uint64_t rb = __ldg(o.row_ptr + qi);
    const uint32_t len = (uint32_t)(__ldg(o.row_ptr + qi + 1) - rb);
    if (len <= (uint32_t)kSortCap)
      warp_query_walk<FLAVOR, CUBE>(t, cx, cy, cz, r, lane, lt, wbuf, kSortCap, nullptr, box);
    warp_row_out<FLAVOR, CUBE>(t, cx, cy, cz, r, lane, lt, wbuf, len, o.cols + rb, rb, o, box);
  } else {
    // single walk into the buffer (count exact even past the buffer)
    const uint32_t cnt =
        warp_query_walk<FLAVOR, CUBE>(t, cx, cy, cz, r, lane, lt, wbuf, kSortCap, nullptr, box);
    unsigned long long base = 0;
    const uint32_t alloc = cnt;
    if (lane == 0) {
      base = atomicAdd(o.cursor, (unsigned long long)alloc);
      if (o.nnz) atomicAdd(o.nnz, (unsigned long long)cnt);
      o.counts[qi] = cnt;
      o.toff[qi] = base;
      o.scnt[qi] = cnt;
    }
    base = __shfl_sync(0xffffffffu, base, 0);
    if (base + alloc <= o.cap) {
      Out o2 = o;
      o2.cur_q = qi;
      warp_row_out<FLAVOR, CUBE>(t, cx, cy, cz, r, lane, lt, wbuf, cnt, o.temp + base, base, o2, box);
    }
  }
}

// Wide query tile: a hull of more than 32 columns (large radii), walked in
// batches of 32 columns — lane c of a batch holds column 32 * batch + c's
// span — with the same staged, warp-uniform record stream and per-lane
// column mask + z window as the compact tile. COUNT / DIGEST keep counters.
// FILL writes each lane's hits UNSORTED at its row (row_ptr from the count
// pass): each lane buffers its hits' handles (u32, kFillCap, stride 33) and
// the warp flushes all buffers, one row at a time (coalesced), whenever one
// could overflow during the next chunk; the rows are sorted afterwards.
template <int FLAVOR, int MODE, int CUBE>
__device__ __forceinline__ void wide_tile(const Tables& t, const Range& R, bool ok, bool active,
                                          uint32_t qi, uint32_t I0, uint32_t J0, uint32_t nj,
                                          uint32_t nc, uint32_t K0, uint32_t K1,
                                          const Predicate& P, int lane, PointRec* stg,
                                          uint32_t* sid, const Out& o,
                                          unsigned long long* wqs) {
  constexpr bool FILL = MODE == MODE_FILL;
  const PointRec* __restrict__ rec = t.rec;
  const uint32_t kk0 = ok ? (uint32_t)R.k0 : 1u;
  const uint32_t kspan = ok ? (uint32_t)(R.k1 - R.k0) : 0u;
  // this lane's own columns, in hull coordinates (an empty range when !ok)
  const uint32_t ri0 = ok ? (uint32_t)R.i0 - I0 : 1u, ri1 = ok ? (uint32_t)R.i1 - I0 : 0u;
  const uint32_t rj0 = ok ? (uint32_t)R.j0 - J0 : 0u, rj1 = ok ? (uint32_t)R.j1 - J0 : 0u;
  uint32_t cnt = 0, ntest = 0, nb = 0, hull = 0;
  uint64_t dig = 0;
  uint64_t wpos = (FILL && active) ? __ldg(o.row_ptr + qi) : 0;
  auto flush = [&]() {
    __syncwarp();
#pragma unroll 4
    for (int l = 0; l < 32; ++l) {
      const uint32_t n = __shfl_sync(0xffffffffu, nb, l);
      const uint64_t wp = __shfl_sync(0xffffffffu, wpos, l);
      CM_DCHECK(n <= (uint32_t)kFillCap + 1u);
      const uint32_t a = (uint32_t)lane < n ? sid[lane * 33 + l] : 0u;
      const uint32_t b2 = lane + 32u < n ? sid[(lane + 32) * 33 + l] : 0u;
      if ((uint32_t)lane < n) o.cols[wp + lane] = a;
      if (lane + 32u < n) o.cols[wp + 32 + lane] = b2;
    }
    wpos += nb;
    nb = 0;
    __syncwarp();
  };
  for (uint32_t cb = 0; cb < nc; cb += 32) {
    const uint32_t col = cb + lane;
    uint32_t b = 0, e = 0;
    if (col < nc) column_span<FLAVOR>(t, I0 + col / nj, J0 + col % nj, K0, K1, &b, &e);
    hull += e - b;
    uint32_t colmask = 0;
    for (uint32_t ci = ri0; ci <= ri1; ++ci) {
      const int64_t lo = (int64_t)ci * nj + rj0 - cb, hi = (int64_t)ci * nj + rj1 - cb;
      if (hi < 0 || lo > 31) continue;
      const uint32_t l2 = lo < 0 ? 0u : (uint32_t)lo, h2 = hi > 31 ? 31u : (uint32_t)hi;
      colmask |= (uint32_t)((((uint64_t)2 << (h2 - l2)) - 1ull) << l2);
    }
    uint32_t needmask = colmask;
#pragma unroll
    for (int sh = 16; sh > 0; sh >>= 1) needmask |= __shfl_xor_sync(0xffffffffu, needmask, sh);
    needmask &= __ballot_sync(0xffffffffu, e > b);
    uint32_t c = 0, p = 0, ce = 0;
    bool more = advance_chunk(needmask, c, p, ce, b, e, true);
    int buf = 0;
    if (more) stage_chunk(stg, rec, p, min(32u, ce - p), lane);
    cp_async_commit();
    while (more) {
      uint32_t c2 = c, p2 = p, ce2 = ce;
      const bool more2 = advance_chunk(needmask, c2, p2, ce2, b, e, false);
      if (more2) stage_chunk(stg + (buf ^ 1) * 32, rec, p2, min(32u, ce2 - p2), lane);
      cp_async_commit();
      cp_async_wait<1>();
      __syncwarp();
      const SRec* sr = reinterpret_cast<const SRec*>(stg + buf * 32);
      const uint32_t len = min(32u, ce - p);
      const bool need = (colmask >> c) & 1u;
      // chunks (k-sorted) outside every lane's z window are skipped whole
      const bool want = need & (sr[len - 1].meta >= kk0) & (sr[0].meta <= kk0 + kspan);
      const bool anyw = __any_sync(0xffffffffu, want);
      if (FILL && anyw && __any_sync(0xffffffffu, nb > (uint32_t)kFillCap - 32u)) flush();
      uint32_t u = anyw ? 0u : len;
      for (; u + 8 <= len; u += 8) {
        SRec v[8];
#pragma unroll
        for (int w = 0; w < 8; ++w) v[w] = sr[u + w];
#pragma unroll
        for (int w = 0; w < 8; ++w) {
          const bool in = need & (v[w].meta - kk0 <= kspan);
          const bool hit = in & pred<CUBE>(P, v[w].x, v[w].y, v[w].z);
          if (MODE == MODE_DIGEST && hit) dig += mix64(v[w].id);
          if (FILL) {
            sid[nb * 33 + lane] = v[w].id;
            nb += hit;
          }
          cnt += hit;
          ntest += in;
        }
      }
      for (; u < len; ++u) {
        const SRec v = sr[u];
        const bool in = need & (v.meta - kk0 <= kspan);
        const bool hit = in & pred<CUBE>(P, v.x, v.y, v.z);
        if (MODE == MODE_DIGEST && hit) dig += mix64(v.id);
        if (FILL) {
          sid[nb * 33 + lane] = v.id;
          nb += hit;
        }
        cnt += hit;
        ntest += in;
      }
      __syncwarp();
      buf ^= 1;
      c = c2, p = p2, ce = ce2;
      more = more2;
    }
    cp_async_wait<0>();
  }
  if (FILL) flush();
  CM_DCHECK(!FILL || !active || wpos == __ldg(o.row_ptr + qi + 1));
  const uint32_t hsum = warp_incl_scan(hull);
  const uint32_t htot = __shfl_sync(0xffffffffu, hsum, 31);
  if (lane == 0) QSTAT_ADD((FILL ? 4 : 0) + 2, htot);
  if (MODE == MODE_COUNT) {
    uint32_t sum = ntest;
#pragma unroll
    for (int sh = 16; sh > 0; sh >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, sh);
    if (lane == 0) QSTAT_ADD(3, sum);
    if (active) {
      if (o.counts) o.counts[qi] = cnt;
      if (o.tested) o.tested[qi] = ntest;
    }
  } else if (MODE == MODE_DIGEST) {
    if (active) {
      o.counts[qi] = cnt;
      o.digests[qi] = dig;
    }
  }
}

// Query-tile kernel (see the file comment).
// XQ: explicit per-centre queries (a radius per centre, kNN brackets, or a
// kernel box per centre, cm_kernel_search). The common batch (one radius,
// centre +- r) is compiled without them: the extra live radius and box
// pointer cost the FILL walk its register budget (spills: wide FILL 34 ->
// 41 ms per launch at r = 2.5).
template <int FLAVOR, int MODE, int CUBE, bool XQ = false>
__global__ void __launch_bounds__(kQThreads, MODE == MODE_FILL ? CM_FILL_MINB
                                             : CUBE == 1 ? CM_CUBE_MINB : CM_QTILE_MINB)
    radius_tile_kernel(
    const Tables t, const double* __restrict__ q, uint64_t nq, double r,
    const uint32_t* __restrict__ perm, const Out o) {
  extern __shared__ __align__(16) unsigned char smraw[];
  constexpr bool ROWS = MODE == MODE_FILL || MODE == MODE_COLLECT;
  constexpr bool FILTERED = CM_FILTER && (CUBE == 0 || CUBE == 1);
  constexpr int so = ROWS ? 4 : 0;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  unsigned char* wreg = smraw + (size_t)wib * warp_smem_bytes<MODE>();
#if CM_QSTATS
  __shared__ unsigned long long s_qs[kQWarps][8];  // this warp's tile counters (QSTAT_ADD)
  unsigned long long* wqs = s_qs[wib];
  if (lane < 8) wqs[lane] = 0ull;
  __syncwarp();
#else
  // (not even declared: 256 bytes of static shared memory moved the collect's
  // shared-memory carve-out and cost it 1.7 %)
  unsigned long long* wqs = nullptr;
#endif
  uint16_t* skey = reinterpret_cast<uint16_t*>(wreg);  // hit = column << 11 | offset in span
  uint32_t* wbuf = reinterpret_cast<uint32_t*>(wreg);
  PointRec* stg = reinterpret_cast<PointRec*>(wreg + row_area_bytes<MODE>());
  const uint32_t lt = lanemask_lt();
  const uint64_t ntiles = (nq + 31) / 32;
  const uint64_t W = (uint64_t)gridDim.x * kQWarps;
  const bool small_grid = t.g.nx < (1ull << 31) && t.g.ny < (1ull << 31) && t.g.nz < (1ull << 31);
  const PointRec* __restrict__ rec = t.rec;

  for (uint64_t tile = (uint64_t)blockIdx.x * kQWarps + wib; tile < ntiles; tile += W) {
    const uint64_t s = tile * 32 + lane;
    const bool active = s < nq;
    constexpr bool SPLIT = MODE == MODE_COLLECT && CM_TILE_SPLIT;
    // COLLECT: a tile whose hull exceeds 32 columns (a sparse query set: the
    // chunks of the host-buffer pipeline, random centre samples) is answered
    // in PARTS — the lower half of the lanes still open, halved again while
    // its hull is too wide — each part by the compact tile walk with the
    // other lanes masked out, instead of one query per warp for all 32
    // lanes. Every other mode keeps one part (wide tiles cover them).
    // (The centre and its range are loaded and derived again for every part, so
    // nothing of them stays live through the walk of the common one-part tile.)
    for (uint32_t pending = __ballot_sync(0xffffffffu, active), part = 0; pending; pending &= ~part) {
    part = pending;
    uint32_t qi = 0u;
    double cx = 0.0, cy = 0.0, cz = 0.0;
    if ((pending >> lane) & 1u) {
      if (q == nullptr) {
        // self queries (cm_radius_search_self): centre s of the cell-ordered
        // records, answered into row rec[s].id — the order the key sort
        // would produce (same keys, both stable by handle)
        const PointRec pr = rec[s];
        qi = pr.id, cx = pr.x, cy = pr.y, cz = pr.z;
      } else {
        qi = __ldg(perm + s);
        cx = __ldg(q + 3 * (uint64_t)qi);
        cy = __ldg(q + 3 * (uint64_t)qi + 1);
        cz = __ldg(q + 3 * (uint64_t)qi + 2);
      }
    }
    // the centre's own radius (kNN radius brackets), else the batch's
    const double rl = (XQ && o.rq && active) ? __ldg(o.rq + qi) : r;
    // explicit kernel boxes (cm_kernel_search: Aabb boxes, bounded cylinders)
    const double* qb = (XQ && o.qbox && active) ? o.qbox + 6 * (uint64_t)qi : nullptr;
    Range R{};
    const bool ok = ((pending >> lane) & 1u) && clamped_range(t.g, cx, cy, cz, rl, &R, CUBE, qb);
    bool act = active, okp = ok;
    bool use_tile = false;
    bool wide = false;
    uint32_t I0 = 0, J0 = 0, nj = 0, ncol = 0, total = 0, K0 = 0, K1 = 0;
    uint64_t nc = 0;
    uint32_t b = 0, e = 0;
    uint32_t I1 = 0, J1 = 0;
    for (;;) {
      const bool inpart = (part >> lane) & 1u;
      act = active && inpart;
      okp = ok && inpart;
      use_tile = small_grid && __any_sync(0xffffffffu, okp);
      if (!use_tile) break;
      I0 = warp_min_u32(okp ? (uint32_t)R.i0 : 0xffffffffu);
      I1 = warp_max_u32(okp ? (uint32_t)R.i1 : 0u);
      J0 = warp_min_u32(okp ? (uint32_t)R.j0 : 0xffffffffu);
      J1 = warp_max_u32(okp ? (uint32_t)R.j1 : 0u);
      nj = J1 - J0 + 1;
      nc = (uint64_t)(I1 - I0 + 1) * nj;
      if (SPLIT && nc > 32 && __popc(part) > CM_TILE_SPLIT_MIN) {
        // keep the lower half of the part's lanes: cut at the lane whose
        // rank within the part is n / 2
        const uint32_t rank = __popc(part & ((2u << lane) - 1u));
        const uint32_t cut = __ballot_sync(0xffffffffu, inpart && rank == (uint32_t)__popc(part) / 2u);
        part &= (2u << (__ffs(cut) - 1)) - 1u;
        continue;
      }
      break;
    }
    if (use_tile) {
      K0 = warp_min_u32(okp ? (uint32_t)R.k0 : 0xffffffffu);
      K1 = warp_max_u32(okp ? (uint32_t)R.k1 : 0u);
      use_tile = nc <= 32;
      if (!use_tile && !o.no_wide && MODE != MODE_COLLECT && (MODE != MODE_FILL || o.wide_fill) &&
          nc <= (uint64_t)kWideMaxCols) {
        // worth it while the lanes' own columns cover >= 1/8 of the hull on average
        uint32_t own = okp ? (uint32_t)((R.i1 - R.i0 + 1) * (R.j1 - R.j0 + 1)) : 0u;
#pragma unroll
        for (int sh = 16; sh > 0; sh >>= 1) own += __shfl_xor_sync(0xffffffffu, own, sh);
        wide = (uint64_t)own * 8 >= nc * 32;
      }
      if (use_tile) {
        ncol = (uint32_t)nc;
        if ((uint32_t)lane < ncol)
          column_span<FLAVOR>(t, I0 + lane / nj, J0 + lane % nj, K0, K1, &b, &e);
        CM_DCHECK(b <= e && e <= t.n);
        total = __shfl_sync(0xffffffffu, warp_incl_scan(e - b), 31);
        // row keys hold a 11-bit offset within a column span
        if (ROWS && warp_max_u32(e - b) > 2048u) use_tile = false;
      }
    }
    if (lane == 0) {
      QSTAT_ADD(so + 0, 1ull);
      if (use_tile) QSTAT_ADD(so + 2, total);
      else if (!wide) QSTAT_ADD(so + 1, 1ull);
    }
    if (wide) {
      Predicate P;
      P.init(cx, cy, cz, rl, CUBE, qb);
      wide_tile<FLAVOR, MODE, CUBE>(t, R, okp, act, qi, I0, J0, nj, (uint32_t)nc, K0, K1, P,
                                    lane, stg, reinterpret_cast<uint32_t*>(wreg), o, wqs);
      __syncwarp();
      continue;
    }
    if (!use_tile) {
      const uint32_t am = __ballot_sync(0xffffffffu, act);
      for (uint32_t lr = am; lr; lr &= lr - 1) {
        const int l = __ffs(lr) - 1;
        const uint32_t ql = __shfl_sync(0xffffffffu, qi, l);
        const double xl = __shfl_sync(0xffffffffu, cx, l);
        const double yl = __shfl_sync(0xffffffffu, cy, l);
        const double zl = __shfl_sync(0xffffffffu, cz, l);
        const double rl2 = __shfl_sync(0xffffffffu, rl, l);
        single_query<FLAVOR, MODE, CUBE>(t, ql, tile * 32 + l, xl, yl, zl, rl2, lane, lt, o, wbuf);
      }
      continue;
    }
    // this lane's columns within the hull, and its k window
    uint32_t colmask = 0;
    if (okp) {
      const uint64_t rowbits = ((1ull << ((uint32_t)(R.j1 - R.j0) + 1)) - 1ull) << ((uint32_t)R.j0 - J0);
      for (uint32_t ci = (uint32_t)R.i0 - I0; ci <= (uint32_t)R.i1 - I0; ++ci)
        colmask |= (uint32_t)(rowbits << (ci * nj));
    }
    const uint32_t kk0 = okp ? (uint32_t)R.k0 : 1u;
    const uint32_t kspan = okp ? (uint32_t)(R.k1 - R.k0) : 0u;
    Predicate P;
    P.init(cx, cy, cz, rl, CUBE, qb);
    uint32_t cnt = 0, ntest = 0;
    uint64_t dig = 0;
    // ROWS: the lane's next key slot as a running shared-memory address
    // (slot i of lane l at 2 * (33 i + l)); advancing it on a hit replaces the
    // per-record slot-address arithmetic, and the row length is recovered
    // from it after the walk
    const uint32_t kaddr0 = ROWS ? (uint32_t)__cvta_generic_to_shared(skey + lane) : 0u;
    const uint32_t klim = kaddr0 + 66u * (uint32_t)kLaneRowCap;
    uint32_t kaddr = kaddr0;
    uint32_t needmask = colmask;
#pragma unroll
    for (int sh = 16; sh > 0; sh >>= 1) needmask |= __shfl_xor_sync(0xffffffffu, needmask, sh);
    uint32_t c = 0, p = 0, ce = 0;
    bool more = advance_chunk(needmask, c, p, ce, b, e, true);
    int buf = 0;
    if (FILTERED && !o.qbox) {
      // Filtered predicates (filter.cuh): fp32 records decide every hit and
      // miss they can prove; the rest go through the exact fp64 test.
      Filter F;
      filter_init<CUBE>(F, t.g, cx, cy, cz, rl,
                        eps_of(t.g, cx, cy, cz, I0, nc / nj, J0, nj));
      // lane l < ncol: corner of hull column l
      const double ccx = col_corner(t.g.ox, I0 + lane / nj, t.g.sx);
      const double ccy = col_corner(t.g.oy, J0 + lane % nj, t.g.sy);
      FRec* stf = reinterpret_cast<FRec*>(stg);
      const FRec* __restrict__ frec = t.frec;
      if (more) stage_chunk_f(stf, frec, p, min(32u, ce - p), lane);
      cp_async_commit();
      while (more) {
        uint32_t c2 = c, p2 = p, ce2 = ce;
        const bool more2 = advance_chunk(needmask, c2, p2, ce2, b, e, false);
        if (more2) stage_chunk_f(stf + (buf ^ 1) * 32, frec, p2, min(32u, ce2 - p2), lane);
        cp_async_commit();
        const float ax = __double2float_rn(__dsub_rn(__shfl_sync(0xffffffffu, ccx, c), F.cx));
        const float ay = __double2float_rn(__dsub_rn(__shfl_sync(0xffffffffu, ccy, c), F.cy));
        cp_async_wait<1>();
        __syncwarp();
        const FRec* sr = stf + buf * 32;
        const uint32_t len = min(32u, ce - p);
        const bool need = (colmask >> c) & 1u;
        const uint32_t kbase = (c << 11) | (p - __shfl_sync(0xffffffffu, b, c));
        // chunks (k-sorted) outside every lane's z window are skipped whole
        const bool want = need & (sr[len - 1].k >= kk0) & (sr[0].k <= kk0 + kspan);
        uint32_t u = __any_sync(0xffffffffu, want) ? 0u : len;
        // a hit at chunk position pos, or nothing (branch-free: a divergent
        // branch here leaves the warp split, and every later shuffle / vote
        // then takes the compiler's WARPSYNC.COLLECTIVE path)
        auto take = [&](uint32_t pos, bool hit) {
          if (MODE == MODE_DIGEST) {
            const uint64_t m = mix64(__ldg(t.ids + p + pos));  // warp-uniform address
            dig += hit ? m : 0ull;
          }
          if (ROWS) {
            sts_u16_if(kaddr, kbase + pos, hit & (kaddr < klim));
            kaddr += hit ? 66u : 0u;
          } else {
            cnt += hit;
          }
        };
        auto resolve = [&](uint32_t unc, uint32_t at) {  // exact fp64 test of the undecided
          if (__any_sync(0xffffffffu, unc != 0u)) {
            Predicate P;
            P.init(F.cx, F.cy, cz, rl, CUBE, nullptr);
            for (int w = 0; w < 8; ++w) {
              if (!__any_sync(0xffffffffu, (unc >> w) & 1u)) continue;
              const PointRec pr = load_rec(rec + p + at + w);  // warp-uniform address
              take(at + w, ((unc >> w) & 1u) && pred<CUBE>(P, pr.x, pr.y, pr.z));
            }
          }
        };
        for (; u + 8 <= len; u += 8) {
          FRec v[8];
#pragma unroll
          for (int w = 0; w < 8; ++w) v[w] = sr[u + w];
          uint32_t unc = 0;
#pragma unroll
          for (int w = 0; w < 8; ++w) {
            const bool in = need & (v[w].k - kk0 <= kspan);
            const float f = filter_value<CUBE>(__fadd_rn(v[w].x, ax), __fadd_rn(v[w].y, ay),
                                               __fadd_rn(v[w].z, F.az));
            const bool hit = in & (f <= F.tin);
            unc |= (in & !(f <= F.tin) & (f <= F.tout)) ? (1u << w) : 0u;
            take(u + w, hit);
            ntest += in;
          }
          resolve(unc, u);
        }
        {
          uint32_t unc = 0;
          const uint32_t u0 = u;
          for (; u < len; ++u) {
            const FRec v = sr[u];
            const bool in = need & (v.k - kk0 <= kspan);
            const float f = filter_value<CUBE>(__fadd_rn(v.x, ax), __fadd_rn(v.y, ay),
                                               __fadd_rn(v.z, F.az));
            const bool hit = in & (f <= F.tin);
            unc |= (in & !(f <= F.tin) & (f <= F.tout)) ? (1u << (u - u0)) : 0u;
            take(u, hit);
            ntest += in;
          }
          resolve(unc, u0);
        }
        __syncwarp();
        buf ^= 1;
        c = c2, p = p2, ce = ce2;
        more = more2;
      }
    } else {
    if (more) stage_chunk(stg, rec, p, min(32u, ce - p), lane);
    cp_async_commit();
    while (more) {
      uint32_t c2 = c, p2 = p, ce2 = ce;
      const bool more2 = advance_chunk(needmask, c2, p2, ce2, b, e, false);
      if (more2) stage_chunk(stg + (buf ^ 1) * 32, rec, p2, min(32u, ce2 - p2), lane);
      cp_async_commit();
      cp_async_wait<1>();
      __syncwarp();
      const SRec* sr = reinterpret_cast<const SRec*>(stg + buf * 32);
      const uint32_t len = min(32u, ce - p);
      const bool need = (colmask >> c) & 1u;
      const uint32_t kbase = (c << 11) | (p - __shfl_sync(0xffffffffu, b, c));
      // chunks (k-sorted) outside every lane's z window are skipped whole
      const bool want = need & (sr[len - 1].meta >= kk0) & (sr[0].meta <= kk0 + kspan);
      uint32_t u = __any_sync(0xffffffffu, want) ? 0u : len;
      // records per group, all loaded before the first test: 8, or 4 for the
      // cube, whose six live bounds otherwise push ptxas into keeping the
      // comparison results in a general register (collect 15.8 -> 18.2 ms)
      constexpr int G = CUBE == 1 ? CM_CUBE_GROUP : 8;
      for (; u + G <= len; u += G) {
        SRec v[G];
#pragma unroll
        for (int w = 0; w < G; ++w) v[w] = sr[u + w];
#pragma unroll
        for (int w = 0; w < G; ++w) {
          const bool in = need & (v[w].meta - kk0 <= kspan);
          const bool hit = in & pred<CUBE>(P, v[w].x, v[w].y, v[w].z);
          if (MODE == MODE_DIGEST && hit) dig += mix64(v[w].id);
          if (ROWS) {
            if (hit && kaddr < klim)
              asm volatile("st.shared.u16 [%0], %1;" ::"r"(kaddr), "h"((unsigned short)(kbase + u + w)));
            kaddr += hit ? 66u : 0u;
          } else {
            cnt += hit;
          }
          ntest += in;
        }
      }
      for (; u < len; ++u) {
        const SRec v = sr[u];
        const bool in = need & (v.meta - kk0 <= kspan);
        const bool hit = in & pred<CUBE>(P, v.x, v.y, v.z);
        if (MODE == MODE_DIGEST && hit) dig += mix64(v.id);
        if (ROWS) {
          if (hit && kaddr < klim)
            asm volatile("st.shared.u16 [%0], %1;" ::"r"(kaddr), "h"((unsigned short)(kbase + u)));
          kaddr += hit ? 66u : 0u;
        } else {
          cnt += hit;
        }
        ntest += in;
      }
      __syncwarp();
      buf ^= 1;
      c = c2, p = p2, ce = ce2;
      more = more2;
    }
    }
    cp_async_wait<0>();
    if (ROWS) cnt = (kaddr - kaddr0) / 66u;
    if (MODE == MODE_COUNT) {
      uint32_t sum = ntest;
#pragma unroll
      for (int sh = 16; sh > 0; sh >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, sh);
      if (lane == 0) QSTAT_ADD(3, sum);
      if (act) {
        if (o.counts) o.counts[qi] = cnt;
        if (o.tested) o.tested[qi] = ntest;
      }
    } else if (MODE == MODE_DIGEST) {
      if (act) {
        o.counts[qi] = cnt;
        o.digests[qi] = dig;
      }
    } else {
      // rows: lanes whose hits overflowed the buffer are redone per query.
      // Their centres wait in the idle staging buffer (bytes 128..1151, past
      // the column starts), so no registers stay live across the row sorts.
      const bool longrow = cnt > (uint32_t)kLaneRowCap;
      uint32_t* spark = reinterpret_cast<uint32_t*>(stg) + 32;
      double* sc = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(stg) + 256);
      if (__any_sync(0xffffffffu, act && longrow)) {
        // the centre and its radius are loaded again here (opaque loads)
        // rather than kept in registers through the walk, where they are
        // dead for the cube: the walk's register pressure decides whether
        // ptxas keeps the eight records' comparison results in predicates
        double rx = 0.0, ry = 0.0, rz = 0.0, rr2 = r;
        if (act) {
          const double* src = q == nullptr ? &rec[s].x : q + 3 * (uint64_t)qi;
          rx = ldg_opaque(src), ry = ldg_opaque(src + 1), rz = ldg_opaque(src + 2);
          if (XQ && o.rq) rr2 = ldg_opaque(o.rq + qi);
        }
        spark[lane] = qi;
        sc[lane] = rx, sc[32 + lane] = ry, sc[64 + lane] = rz, sc[96 + lane] = rr2;
      }
      const uint32_t mine = (act && !longrow) ? cnt : 0u;
      uint64_t dst;
      bool write_ok = true;
      if (MODE == MODE_FILL) {
        dst = act ? __ldg(o.row_ptr + qi) : 0;
        // the row the count pass sized must hold exactly this walk's hits
        CM_DCHECK(!act || longrow || __ldg(o.row_ptr + qi + 1) - dst == (uint64_t)cnt);
      } else {
        const uint32_t alloc = mine;
        const uint32_t inc = warp_incl_scan(alloc);
        const uint32_t tot = __shfl_sync(0xffffffffu, inc, 31);
        unsigned long long base = 0;
        if (lane == 0 && tot) {
          base = atomicAdd(o.cursor, (unsigned long long)tot);
          if (o.nnz) atomicAdd(o.nnz, (unsigned long long)tot);
        }
        base = __shfl_sync(0xffffffffu, base, 0);
        dst = base + (inc - alloc);
        write_ok = base + tot <= o.cap;
        CM_DCHECK(!write_ok || dst + alloc <= o.cap);
        if (act && !longrow) {
          o.counts[qi] = cnt;
          o.toff[qi] = dst;
          o.scnt[qi] = cnt;
        }
      }
      __syncwarp();
      uint32_t* rows = MODE == MODE_FILL ? o.cols : o.temp;
      if (write_ok) {
        // hit keys -> handles (the records were just walked: L1/L2 hits)
        __syncwarp();
        if (MODE == MODE_COLLECT) {
          // Arena rows go out unsorted (the gather sorts), so each lane
          // translates and stores its own row: independent loads, many in
          // flight, no warp-wide round trip per row. Column starts move to
          // the (now idle) staging buffer so the loop needs no shuffles.
          // (Sorting here instead — per-lane networks after the walk — put
          // the network's 17 KB of code next to the walk's and the kernel
          // thrashed the 32 KB instruction cache: collect 10.7 -> 22 ms.)
          uint32_t* cbeg = reinterpret_cast<uint32_t*>(stg);
          cbeg[lane] = b;
          __syncwarp();
          uint32_t* out = rows + dst;
          uint32_t i = 0;
          for (; i + 8 <= mine; i += 8) {
            uint32_t kv[8], v[8];
#pragma unroll
            for (int w = 0; w < 8; ++w) kv[w] = skey[(i + w) * 33 + lane];
#pragma unroll
            for (int w = 0; w < 8; ++w) v[w] = __ldg(t.ids + cbeg[kv[w] >> 11] + (kv[w] & 2047u));
#pragma unroll
            for (int w = 0; w < 8; ++w) out[i + w] = v[w];
          }
          for (; i < mine; ++i) {
            const uint32_t kv = skey[i * 33 + lane];
            out[i] = __ldg(t.ids + cbeg[kv >> 11] + (kv & 2047u));
          }
        } else
        for (int l = 0; l < 32; ++l) {
          const uint32_t len = __shfl_sync(0xffffffffu, mine, l);
          const uint64_t off = __shfl_sync(0xffffffffu, dst, l);
          if (len == 0) continue;
          uint32_t v[4];
#pragma unroll
          for (int r2 = 0; r2 < 4; ++r2) {
            const uint32_t i = r2 * 32 + lane;
            const uint32_t key = i < len ? skey[i * 33 + l] : 0u;
            const uint32_t cb2 = __shfl_sync(0xffffffffu, b, key >> 11);
            v[r2] = i < len ? __ldg(t.ids + cb2 + (key & 2047u)) : 0xffffffffu;
          }
          if (MODE == MODE_COLLECT) {  // arena rows go out unsorted; the gather sorts
#pragma unroll
            for (int r2 = 0; r2 < 4; ++r2) {
              const uint32_t i = r2 * 32 + lane;
              if (i < len) rows[off + i] = v[r2];
            }
          } else {
            warp_sort_regs<4>(v, lane);
#pragma unroll
            for (int r2 = 0; r2 < 4; ++r2) {
              const uint32_t i = r2 * 32 + lane;
              if (i < len) rows[off + i] = v[r2];
            }
          }
        }
      }
      __syncwarp();
      const uint32_t lm = __ballot_sync(0xffffffffu, act && longrow);
      if (lane == 0 && lm) QSTAT_ADD(7, __popc(lm));
      // single_query reuses the whole warp region: take every parked centre
      // into registers first (lane l holds centre l)
      uint32_t pq = qi;
      double px = 0.0, py = 0.0, pz = 0.0, pr = r;
      if (lm) {  // warp-uniform; the loads are branch-free selects
        const bool mine = (lm >> lane) & 1u;
        const uint32_t a = spark[lane];
        const double b0 = sc[lane], b1 = sc[32 + lane], b2 = sc[64 + lane], b3 = sc[96 + lane];
        pq = mine ? a : pq;
        px = mine ? b0 : px, py = mine ? b1 : py, pz = mine ? b2 : pz, pr = mine ? b3 : pr;
      }
      __syncwarp();
      for (uint32_t lr = lm; lr; lr &= lr - 1) {
        const int l = __ffs(lr) - 1;
        const uint32_t ql = __shfl_sync(0xffffffffu, pq, l);
        const double xl = __shfl_sync(0xffffffffu, px, l);
        const double yl = __shfl_sync(0xffffffffu, py, l);
        const double zl = __shfl_sync(0xffffffffu, pz, l);
        const double rl2 = __shfl_sync(0xffffffffu, pr, l);
        single_query<FLAVOR, MODE, CUBE>(t, ql, tile * 32 + l, xl, yl, zl, rl2, lane, lt, o, wbuf);
      }
    }
    __syncwarp();
    }  // parts
  }
#if CM_QSTATS
  __syncwarp();
  if (lane < 8 && wqs[lane]) atomicAdd(&g_qstats[lane], wqs[lane]);
#endif
}

// Rows too long for a warp buffer: one block per row (persistent blocks).
__global__ void __launch_bounds__(1024) big_row_sort_kernel(uint32_t* __restrict__ rows,
                                                            const uint64_t* __restrict__ big_off,
                                                            const uint32_t* __restrict__ big_len,
                                                            const uint32_t* __restrict__ n_big) {
  extern __shared__ uint32_t sm[];
  const uint32_t nb = *n_big;
  for (uint32_t bi = blockIdx.x; bi < nb; bi += gridDim.x) {
    uint32_t* row = rows + big_off[bi];
    const uint32_t len = big_len[bi];
    if (len <= (uint32_t)kBigSmemCap) {
      for (uint32_t x = threadIdx.x; x < len; x += blockDim.x) sm[x] = row[x];
      __syncthreads();
      bitonic_sort(sm, len, threadIdx.x, blockDim.x, [] { __syncthreads(); });
      for (uint32_t x = threadIdx.x; x < len; x += blockDim.x) row[x] = sm[x];
    } else {
      bitonic_sort(row, len, threadIdx.x, blockDim.x, [] { __syncthreads(); });
    }
    __syncthreads();
  }
}

// Rows of 97..1024 handles, one warp per row, blocked layout: lane l holds
// handles [l * ITEMS, (l + 1) * ITEMS) of the row in registers, so the
// bitonic network's exchanges at distance < ITEMS stay inside a lane (no
// shuffles) and the row's loads and stores are contiguous per lane.
constexpr int kBlockedMax = 1024;
#ifndef CM_MID_MIN
#define CM_MID_MIN 1024
#endif
constexpr int kMidMin = CM_MID_MIN;  // rows above this go to sort_mid_rows_kernel

template <int ITEMS>
__device__ __forceinline__ void warp_sort_blocked(uint32_t (&v)[ITEMS], int lane) {
  constexpr int P = 32 * ITEMS;
#pragma unroll
  for (int k = 2; k <= P; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j < ITEMS) {
#pragma unroll
        for (int r = 0; r < ITEMS; ++r) {
          const int p = r ^ j;
          if (p > r) {
            const bool asc = (((uint32_t)lane * ITEMS + r) & k) == 0;
            const uint32_t a = v[r], b = v[p];
            v[r] = asc ? min(a, b) : max(a, b);
            v[p] = asc ? max(a, b) : min(a, b);
          }
        }
      } else {
        const int jl = j / ITEMS;
        const bool lower = (lane & jl) == 0;
#pragma unroll
        for (int r = 0; r < ITEMS; ++r) {
          const uint32_t o = __shfl_xor_sync(0xffffffffu, v[r], jl);
          const bool asc = (((uint32_t)lane * ITEMS + r) & k) == 0;
          v[r] = (lower == asc) ? min(v[r], o) : max(v[r], o);
        }
      }
    }
  }
}

template <int ITEMS>
__device__ __forceinline__ void warp_sort_row_blocked(uint32_t* row, uint32_t n, int lane) {
  uint32_t v[ITEMS];
#pragma unroll
  for (int r = 0; r < ITEMS; ++r) {
    const uint32_t e = (uint32_t)lane * ITEMS + r;
    v[r] = e < n ? row[e] : 0xffffffffu;
  }
  warp_sort_blocked<ITEMS>(v, lane);
#pragma unroll
  for (int r = 0; r < ITEMS; ++r) {
    const uint32_t e = (uint32_t)lane * ITEMS + r;
    if (e < n) row[e] = v[r];
  }
}

// Arena rows -> CSR order, sorting them on the way. A warp takes 32
// consecutive queries in the caller's order, so its output is one contiguous
// stretch of cols (whole sectors, no partial-sector read-modify-write in L2);
// the arena rows it reads are scattered but each is a short burst. Rows of <= 96
// handles are staged in shared memory (interleaved, stride 33); each lane
// sorts its own row in registers with an unrolled bitonic network — rows
// longer than 64 as two runs, [0, 64) and [64, len), merged by the warp
// along the merge path (three outputs per lane). Rows of 97..128 (tile rows
// past the staging width) are sorted by the warp (blocked register bitonic);
// longer ones come from the one-query-per-warp path already sorted and are
// copied.
#ifndef CM_GATHER_ROW
#define CM_GATHER_ROW 96
#endif
constexpr int kGatherRow = CM_GATHER_ROW;
#ifndef CM_GATHER_NET16
#define CM_GATHER_NET16 0  // 16-wide network for short groups: one more network in the i-cache (gather 5.99 -> 6.08 ms)
#endif
static_assert(kGatherRow > 64 && kGatherRow <= 96, "gather staging: run 1 of 64 + run 2 <= 32");
constexpr int kGatherWarpWords = kGatherRow * 33 + 96;  // rows, sfin[32], srel[32] (u64)
//
// SORT = true is the in-place row sort after a wide-tile FILL (temp == cols,
// toff == row_ptr, lengths from row_ptr): only rows <= 96 are handled here;
// longer rows are sorted by sort_mid_rows_kernel / big_row_sort_kernel.
template <bool SORT>
#ifdef CM_GATHER_MINB
#define CM_GATHER_BOUNDS __launch_bounds__(128, CM_GATHER_MINB)
#else
#define CM_GATHER_BOUNDS __launch_bounds__(128)
#endif
__global__ void CM_GATHER_BOUNDS gather_rows_kernel(const uint32_t* temp,
                                                          const uint64_t* __restrict__ toff,
                                                          const uint32_t* __restrict__ counts,
                                                          const uint64_t* __restrict__ row_ptr,
                                                          uint32_t* cols, uint64_t nq,
                                                          uint32_t skip_above = 0xffffffffu) {
  extern __shared__ uint32_t gsm[];
  const int lane = threadIdx.x & 31;
  uint32_t* srow = gsm + (threadIdx.x >> 5) * kGatherWarpWords;
  uint32_t* sfin = srow + kGatherRow * 33;                          // flat row ends
  uint64_t* srel = reinterpret_cast<uint64_t*>(sfin + 32);           // row starts - row 0's
  const uint64_t ngroups = (nq + 31) / 32;
  const uint64_t W = (uint64_t)gridDim.x * (blockDim.x >> 5);
  uint64_t gidx = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  uint32_t nlen = 0;
  uint64_t nso = 0;
  auto row_len = [&](uint64_t qq) -> uint32_t {
    return SORT ? (uint32_t)(__ldg(row_ptr + qq + 1) - __ldg(row_ptr + qq)) : __ldg(counts + qq);
  };
  if (gidx < ngroups && gidx * 32 + lane < nq) {
    nlen = row_len(gidx * 32 + lane);
    nso = __ldg(toff + gidx * 32 + lane);
  }
  for (; gidx < ngroups; gidx += W) {
    const uint64_t q = gidx * 32 + lane;
    const bool act = q < nq;
    const uint32_t len = nlen;
    const uint64_t so = nso;
    const uint64_t dof = act ? __ldg(row_ptr + q) : 0;
    CM_DCHECK(!act || __ldg(row_ptr + q + 1) - dof == (uint64_t)len);
    // the next group's arena rows start moving into L2 while this one sorts
    {
      const uint64_t nq2 = (gidx + W) * 32 + lane;
      nlen = 0, nso = 0;
      if (nq2 < nq) {
        nlen = row_len(nq2);
        nso = __ldg(toff + nq2);
        if (nlen <= (uint32_t)kGatherRow) {
          const char* a = reinterpret_cast<const char*>(temp + nso);
          const char* e = reinterpret_cast<const char*>(temp + nso + nlen);
          for (const char* x = reinterpret_cast<const char*>((uintptr_t)a & ~(uintptr_t)127); x < e; x += 128)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(x));
        }
      }
    }
    const uint32_t staged = len <= (uint32_t)kGatherRow ? len : 0u;
    // 8 rows per step, all their loads in flight before the stores
    for (int l0 = 0; l0 < 32; l0 += 8) {
      uint32_t v[8][3];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t ln = __shfl_sync(0xffffffffu, staged, l0 + j);
        const uint64_t o = __shfl_sync(0xffffffffu, so, l0 + j);
#pragma unroll
        for (int h = 0; h < 3; ++h) {
          const uint32_t i = h * 32 + lane;
          v[j][h] = i < ln ? __ldg(temp + o + i) : 0u;
        }
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t ln = __shfl_sync(0xffffffffu, staged, l0 + j);
#pragma unroll
        for (int h = 0; h < 3; ++h) {
          const uint32_t i = h * 32 + lane;
          if (i < ln) srow[i * 33 + l0 + j] = v[j][h];
        }
      }
    }
    __syncwarp();
    // run 1: [0, min(len, 64))
    const uint32_t r1 = staged < 64u ? staged : 64u;
    const uint32_t m1 = warp_max_u32(r1);
    if (m1 > 32) lane_sort_row<64>(srow, lane, r1);
#if CM_GATHER_NET16
    else if (m1 > 16) lane_sort_row<32>(srow, lane, r1);
    else if (m1 > 1) lane_sort_row<16>(srow, lane, r1);
#else
    else if (m1 > 1) lane_sort_row<32>(srow, lane, r1);  // one network less in the i-cache
#endif
    // run 2: [64, len)
    const uint32_t r2 = staged > 64u ? staged - 64u : 0u;
    const uint32_t m2 = warp_max_u32(r2);
    if (m2 > 1) lane_sort_row<(kGatherRow - 64 <= 16 ? 16 : 32)>(srow + 64 * 33, lane, r2);
    __syncwarp();
    // Rows of <= 64 (one sorted run) leave as one flat stream: flat element
    // f belongs to the row whose flat range holds it; every lane walks the
    // small row table forward (rows average fewer than 32 handles per lane
    // step, so the walk is one or two probes).
    {
      const uint32_t flen = len <= 64u ? len : 0u;
      const uint32_t fin = warp_incl_scan(flen);
      const uint32_t ftot = __shfl_sync(0xffffffffu, fin, 31);
      const uint64_t d0 = __shfl_sync(0xffffffffu, dof, 0);
      sfin[lane] = fin;
      srel[lane] = dof - d0;
      __syncwarp();
      uint32_t l = 0, fstart = 0;
      for (uint32_t f = lane; f < ftot; f += 32) {
        uint32_t e = sfin[l];
        while (e <= f) {
          fstart = e;
          e = sfin[++l];
        }
        const uint32_t i = f - fstart;
        cols[d0 + srel[l] + i] = srow[i * 33 + l];
      }
    }
    for (uint32_t lm = __ballot_sync(0xffffffffu, len > 64u && (!SORT || len <= (uint32_t)kGatherRow));
         lm; lm &= lm - 1) {
      const int l = __ffs(lm) - 1;
      const uint32_t ln = __shfl_sync(0xffffffffu, len, l);
      const uint64_t d = __shfl_sync(0xffffffffu, dof, l);
      if (ln <= (uint32_t)kGatherRow) {
        // merge path: lane takes outputs [3 lane, 3 lane + 3) — co-rank of
        // its diagonal by binary search, then three sequential merge steps
        // (handles are distinct, so ties never occur)
        const uint32_t nb = ln - 64;
        const uint32_t* A = srow + l;
        const uint32_t* B = srow + 64 * 33 + l;
        const uint32_t dg = min(3u * (uint32_t)lane, ln);
        uint32_t lo = dg > nb ? dg - nb : 0u, hi = min(dg, 64u);
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (A[mid * 33] < B[(dg - 1 - mid) * 33]) lo = mid + 1; else hi = mid;
        }
        uint32_t ia = lo, ib = dg - lo;
#pragma unroll
        for (int t = 0; t < 3; ++t) {
          if (dg + t < ln) {
            const uint32_t av = ia < 64u ? A[ia * 33] : 0xffffffffu;
            const uint32_t bv = ib < nb ? B[ib * 33] : 0xffffffffu;
            const bool ta = av < bv;
            cols[d + dg + t] = ta ? av : bv;
            ia += ta;
            ib += !ta;
          }
        }
      } else if (!SORT && ln <= (uint32_t)kLaneRowCap) {
        // an unsorted tile row past the staging width: one warp, blocked
        // register bitonic, straight from the arena to the CSR
        const uint64_t o = __shfl_sync(0xffffffffu, so, l);
        uint32_t v[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const uint32_t e = (uint32_t)lane * 4 + r;
          v[r] = e < ln ? __ldg(temp + o + e) : 0xffffffffu;
        }
        warp_sort_blocked<4>(v, lane);
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const uint32_t e = (uint32_t)lane * 4 + r;
          if (e < ln) cols[d + e] = v[r];
        }
      } else if (ln <= skip_above) {  // longer rows: merge_big_rows_kernel wrote them
        const uint64_t o = __shfl_sync(0xffffffffu, so, l);
        for (uint32_t b0 = 0; b0 < ln; b0 += 256) {  // 8 loads in flight per lane
          uint32_t v[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint32_t i = b0 + 32 * j + lane;
            v[j] = i < ln ? __ldg(temp + o + i) : 0u;
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint32_t i = b0 + 32 * j + lane;
            if (i < ln) cols[d + i] = v[j];
          }
        }
      }
    }
    __syncwarp();
  }
}

// One size class per launch (rows of (LO, 32 * ITEMS] handles), so the
// register budget, hence the occupancy, fits the class.
template <int ITEMS>
__global__ void __launch_bounds__(128) sort_blocked_rows_kernel(uint32_t* cols,
                                                                const uint64_t* __restrict__ row_ptr,
                                                                uint64_t nq, uint32_t lo) {
  const int lane = threadIdx.x & 31;
  const uint64_t ngroups = (nq + 31) / 32;
  const uint64_t W = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t g = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); g < ngroups;
       g += W) {
    const uint64_t q = g * 32 + lane;
    uint64_t b = 0;
    uint32_t len = 0;
    if (q < nq) {
      b = __ldg(row_ptr + q);
      len = (uint32_t)(__ldg(row_ptr + q + 1) - b);
    }
    for (uint32_t lm = __ballot_sync(0xffffffffu, len > lo && len <= 32u * ITEMS); lm;
         lm &= lm - 1) {
      const int l = __ffs(lm) - 1;
      const uint32_t n = __shfl_sync(0xffffffffu, len, l);
      warp_sort_row_blocked<ITEMS>(cols + __shfl_sync(0xffffffffu, b, l), n, lane);
    }
  }
}

// Rows of (32 HI, 64 HI] handles, one warp per row, without padding the
// whole row to the next power of two: the head [0, 32 HI) is sorted by the
// blocked register network, the tail [32 HI, n) by the smallest network that
// holds it, and the two runs are merged along the merge path through shared
// memory (each lane: co-rank by binary search, then ceil(n / 32) merge
// steps), then copied back coalesced. Used for 513..1024 (a 512-network,
// a tail network and the merge instead of a 1024-network); for shorter rows
// the padded network measured faster (r = 2.5 fill + sort 95 -> 103 ms when
// 129..512 were split too).
__device__ __forceinline__ uint32_t spad(uint32_t p) { return p + (p >> 5); }

template <int TI>
__device__ __forceinline__ void split_sort_tail(const uint32_t* src, uint32_t t, uint32_t* dst,
                                                int lane) {
  uint32_t v[TI];
#pragma unroll
  for (int r = 0; r < TI; ++r) {
    const uint32_t e = (uint32_t)lane * TI + r;
    v[r] = e < t ? src[e] : 0xffffffffu;
  }
  warp_sort_blocked<TI>(v, lane);
#pragma unroll
  for (int r = 0; r < TI; ++r) {
    const uint32_t e = (uint32_t)lane * TI + r;
    if (e < t) dst[spad(e)] = v[r];
  }
}

template <int HI>
__device__ __forceinline__ void warp_sort_row_split(uint32_t* row, uint32_t n, uint32_t* sa,
                                                    uint32_t* so, int lane) {
  constexpr uint32_t H = 32u * HI;
  const uint32_t t = n - H;  // 1 .. H
  {
    uint32_t v[HI];
#pragma unroll
    for (int r = 0; r < HI; ++r) v[r] = row[(uint32_t)lane * HI + r];
    warp_sort_blocked<HI>(v, lane);
#pragma unroll
    for (int r = 0; r < HI; ++r) sa[spad((uint32_t)lane * HI + r)] = v[r];
  }
  uint32_t* sb = sa + spad(H);  // tail run, its own padded indices
  if (t <= 32) {
    uint32_t v = (uint32_t)lane < t ? row[H + lane] : 0xffffffffu;
    v = warp_sort32(v, lane);
    if ((uint32_t)lane < t) sb[spad(lane)] = v;
  } else if (HI >= 4 && t <= H / 4) {
    split_sort_tail<(HI >= 4 ? HI / 4 : 1)>(row + H, t, sb, lane);
  } else if (HI >= 2 && t <= H / 2) {
    split_sort_tail<(HI >= 2 ? HI / 2 : 1)>(row + H, t, sb, lane);
  } else {
    split_sort_tail<HI>(row + H, t, sb, lane);
  }
  __syncwarp();
  const uint32_t per = (n + 31) >> 5;
  const uint32_t d = min((uint32_t)lane * per, n);
  uint32_t lo = d > t ? d - t : 0u, hi = min(d, H);
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (sa[spad(mid)] <= sb[spad(d - 1 - mid)]) lo = mid + 1; else hi = mid;
  }
  uint32_t ia = lo, ib = d - lo;
  for (uint32_t s2 = 0; s2 < per && d + s2 < n; ++s2) {
    const bool ta = ib >= t || (ia < H && sa[spad(ia)] <= sb[spad(ib)]);
    so[spad(d + s2)] = ta ? sa[spad(ia)] : sb[spad(ib)];
    ia += ta;
    ib += !ta;
  }
  __syncwarp();
  for (uint32_t i = lane; i < n; i += 32) row[i] = so[spad(i)];
  __syncwarp();
}

constexpr int kSplitWarpWords = 2 * (kBlockedMax + kBlockedMax / 32 + 2);

template <int HI>
__global__ void __launch_bounds__(128) sort_split_rows_kernel(uint32_t* cols,
                                                              const uint64_t* __restrict__ row_ptr,
                                                              uint64_t nq) {
  extern __shared__ uint32_t ssm[];
  uint32_t* sa = ssm + (threadIdx.x >> 5) * kSplitWarpWords;
  uint32_t* so = sa + kSplitWarpWords / 2;
  const int lane = threadIdx.x & 31;
  const uint64_t ngroups = (nq + 31) / 32;
  const uint64_t W = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t g = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); g < ngroups;
       g += W) {
    const uint64_t q = g * 32 + lane;
    uint64_t b = 0;
    uint32_t len = 0;
    if (q < nq) {
      b = __ldg(row_ptr + q);
      len = (uint32_t)(__ldg(row_ptr + q + 1) - b);
    }
    for (uint32_t lm = __ballot_sync(0xffffffffu, len > 32u * HI && len <= 64u * HI); lm;
         lm &= lm - 1) {
      const int l = __ffs(lm) - 1;
      const uint32_t n = __shfl_sync(0xffffffffu, len, l);
      warp_sort_row_split<HI>(cols + __shfl_sync(0xffffffffu, b, l), n, sa, so, lane);
    }
  }
}

// In-place sort of the rows of 1025..8192 handles (after a wide-tile FILL;
// shorter rows were sorted by the gather pass and sort_blocked_rows_kernel,
// longer ones are listed for big_row_sort_kernel). A block of 128 threads packs consecutive rows into a
// GROUP of at most 128 runs of 64 handles (row-aligned) and stages it in
// shared memory, each row contiguous from 64 * (its first run), with an XOR
// swizzle (word p at p ^ ((p >> 6) & 31)) so that both the run-per-thread
// and the linear accesses are bank-conflict free. Thread t sorts run t in
// registers (unrolled bitonic), then every row's runs are merged pairwise,
// 64 -> 128 -> ..., along the merge path: each round, thread t produces the
// 64 outputs at its run's position as four independent 16-output streams
// (co-rank by binary search for each; branch-free steps), ping-ponging
// between two buffers. A row stops after ceil(log2(runs)) rounds and is
// written back from whichever buffer holds it.
constexpr int kMidThreads = 128;
constexpr int kMidMax = 64 * kMidThreads;
constexpr int kMidBuf = kMidMax + 64;  // one slot past a row end stays in bounds

__device__ __forceinline__ uint32_t mid_swz(uint32_t p) { return p ^ ((p >> 6) & 31u); }

__global__ void __launch_bounds__(kMidThreads) sort_mid_rows_kernel(
    uint32_t* cols, const uint64_t* __restrict__ row_ptr, uint64_t nq, uint64_t* big_off,
    uint32_t* big_len, uint32_t* n_big, uint32_t mid_min) {
  extern __shared__ uint32_t msm[];
  __shared__ uint32_t s_off[kMidThreads], s_len[kMidThreads], s_rb[kMidThreads],
      s_runs[kMidThreads];
  __shared__ uint32_t s_wsum[kMidThreads / 32], s_wfit[kMidThreads / 32],
      s_wmax[kMidThreads / 32], s_wbig[kMidThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  constexpr uint64_t kTask = 1024;
  const uint64_t ntasks = (nq + kTask - 1) / kTask;
  for (uint64_t task = blockIdx.x; task < ntasks; task += gridDim.x) {
    uint64_t q = task * kTask;
    const uint64_t qend = min(nq, q + kTask);
    while (q < qend) {
      const uint64_t ql = q + tid;
      uint64_t st = 0;
      uint32_t len = 0;
      if (ql < qend) {
        st = __ldg(row_ptr + ql);
        len = (uint32_t)(__ldg(row_ptr + ql + 1) - st);
      }
      const uint32_t runs =
          (len > mid_min && len <= (uint32_t)kMidMax) ? (len + 63) >> 6 : 0u;
      const uint32_t winc = warp_incl_scan(runs);
      // a group ends at the 128-run budget and before the first row past
      // kMidMax (which, when first, forms a group of its own: listed for the
      // block sort), so the group's handles are one short contiguous span
      const uint32_t bigm = __ballot_sync(0xffffffffu, ql < qend && len > (uint32_t)kMidMax);
      if (lane == 31) s_wsum[wid] = winc;
      if (lane == 0) s_wbig[wid] = bigm ? (uint32_t)(wid * 32 + __ffs(bigm) - 1) : 0xffffffffu;
      __syncthreads();
      uint32_t woff = 0, firstbig = 0xffffffffu;
#pragma unroll
      for (int w = 0; w < kMidThreads / 32; ++w) {
        woff += w < wid ? s_wsum[w] : 0u;
        firstbig = min(firstbig, s_wbig[w]);
      }
      const uint32_t rincl = woff + winc;
      const uint32_t cut = firstbig == 0 ? 1u : firstbig;
      const bool fit = ql < qend && rincl <= (uint32_t)kMidThreads && (uint32_t)tid < cut;
      const uint32_t fm = __ballot_sync(0xffffffffu, fit);
      const uint32_t rm = fit ? runs : 0u;
      const uint32_t wmax = warp_max_u32(rm);
      if (lane == 0) s_wfit[wid] = __popc(fm), s_wmax[wid] = wmax;
      const uint32_t big = fm & bigm;
      if (big) {
        uint32_t slot = 0;
        if (lane == 0) slot = atomicAdd(n_big, (uint32_t)__popc(big));
        slot = __shfl_sync(0xffffffffu, slot, 0);
        if ((big >> lane) & 1u) {
          const uint32_t at = slot + __popc(big & lanemask_lt());
          big_off[at] = st;
          big_len[at] = len;
        }
      }
      const uint64_t g0 = __ldg(row_ptr + q);  // the group's first handle
      s_off[tid] = (uint32_t)(st - g0);         // meaningful for the group's rows
      s_len[tid] = len;
      s_rb[tid] = rincl - runs;
      s_runs[tid] = rm;
      __syncthreads();
      uint32_t g = 0, maxruns = 0;
#pragma unroll
      for (int w = 0; w < kMidThreads / 32; ++w) g += s_wfit[w], maxruns = max(maxruns, s_wmax[w]);
      const uint32_t nruns = s_rb[g - 1] + s_runs[g - 1];
      if (nruns) {
        uint32_t* b0 = msm;
        {  // load the group's rows by run slot (slot f = 64 * run + offset,
           // the row's smem position), 8 loads in flight per thread; only the
           // grouped rows' handles are read, not the shorter rows between
           // them (which the earlier span load read and dropped: a second
           // full pass over the CSR when long rows are sparse)
          const uint32_t nslots = 64u * nruns;
          uint32_t r = 0;
          for (uint32_t f0 = 0; f0 < nslots; f0 += 8 * kMidThreads) {
            uint32_t v[8];
            uint32_t ok = 0;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const uint32_t f = f0 + k * kMidThreads + tid;
              v[k] = 0u;
              if (f < nslots) {
                while (r + 1 < g && 64u * s_rb[r + 1] <= f) ++r;
                const uint32_t idx = f - 64u * s_rb[r];
                if (idx < s_len[r]) {
                  v[k] = cols[g0 + s_off[r] + idx];
                  ok |= 1u << k;
                }
              }
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const uint32_t f = f0 + k * kMidThreads + tid;
              if ((ok >> k) & 1u) b0[mid_swz(f)] = v[k];
            }
          }
        }
        __syncthreads();
        // this thread's run: row L = the last row with runs whose rb <= tid
        const bool own = (uint32_t)tid < nruns;
        uint32_t L = 0;
        if (own) {
          uint32_t lo = 0, hi = g - 1;
          while (lo < hi) {
            const uint32_t m = (lo + hi + 1) >> 1;
            if (s_rb[m] <= (uint32_t)tid) lo = m; else hi = m - 1;
          }
          L = lo;
          while (s_runs[L] == 0) --L;
        }
        const uint32_t rl = own ? s_len[L] : 0u;
        const uint32_t base = own ? 64u * s_rb[L] : 0u;
        const uint32_t j = (uint32_t)tid - (own ? s_rb[L] : 0u);
        if (own) {
          const uint32_t n = min(64u, rl - 64u * j);
          uint32_t v[64];
#pragma unroll
          for (int i = 0; i < 64; ++i)
            v[i] = (uint32_t)i < n ? b0[mid_swz(base + 64u * j + i)] : 0xffffffffu;
          lane_sort_regs<64>(v);
#pragma unroll
          for (int i = 0; i < 64; ++i)
            if ((uint32_t)i < n) b0[mid_swz(base + 64u * j + i)] = v[i];
        }
        __syncthreads();
        int cur = 0;
        for (uint32_t w = 64; w < 64u * maxruns; w <<= 1) {
          if (own && w < rl) {  // this row still has runs to merge
            const uint32_t* src = msm + cur * kMidBuf;
            uint32_t* dst = msm + (cur ^ 1) * kMidBuf;
            // outputs [o0, o0 + 64) are one 64-word block: constant swizzle
            uint32_t* dblk = dst + base + 64u * j;
            const uint32_t dsw = (base / 64u + j) & 31u;
            const uint32_t o0 = 64u * j;
            const uint32_t pb = o0 / (2 * w) * (2 * w);
            const uint32_t a1 = min(pb + w, rl), b1 = min(pb + 2 * w, rl);
            const uint32_t na = a1 - pb, nb = b1 - a1;
            const uint32_t A0 = base + pb, B0 = base + a1;
            uint32_t ia[4], ib[4], av[4], bv[4];
#pragma unroll
            for (int s4 = 0; s4 < 4; ++s4) {
              const uint32_t dd = min(o0 + 16u * s4, rl) - pb;
              uint32_t lo = dd > nb ? dd - nb : 0u, hi = min(dd, na);
              while (lo < hi) {
                const uint32_t m = (lo + hi) >> 1;
                if (src[mid_swz(A0 + m)] < src[mid_swz(B0 + dd - 1 - m)]) lo = m + 1; else hi = m;
              }
              ia[s4] = lo;
              ib[s4] = dd - lo;
              const uint32_t x = src[mid_swz(A0 + lo)], y = src[mid_swz(B0 + dd - lo)];
              av[s4] = lo < na ? x : 0xffffffffu;
              bv[s4] = dd - lo < nb ? y : 0xffffffffu;
            }
            const uint32_t oend = min(o0 + 64u, rl);
#pragma unroll 2
            for (int step = 0; step < 16; ++step) {
#pragma unroll
              for (int s4 = 0; s4 < 4; ++s4) {
                const uint32_t o = o0 + 16u * s4 + step;
                const bool ta = av[s4] < bv[s4];  // handles are distinct
                if (o < oend) dblk[(16u * s4 + step) ^ dsw] = ta ? av[s4] : bv[s4];
                ia[s4] += ta;
                ib[s4] += !ta;
                const uint32_t idx = ta ? A0 + ia[s4] : B0 + ib[s4];
                const bool more = ta ? ia[s4] < na : ib[s4] < nb;
                const uint32_t nv = src[mid_swz(idx)];
                const uint32_t nv2 = more ? nv : 0xffffffffu;
                av[s4] = ta ? nv2 : av[s4];
                bv[s4] = ta ? bv[s4] : nv2;
              }
            }
          }
          cur ^= 1;
          __syncthreads();
        }
        {  // write back: a row with R runs ended in buffer (ceil(log2 R) & 1)
          uint32_t r = 0;
          for (uint32_t f = tid; f < 64u * nruns; f += kMidThreads) {
            while (r + 1 < g && 64u * s_rb[r + 1] <= f) ++r;
            const uint32_t idx = f - 64u * s_rb[r];
            if (idx < s_len[r]) {
              const uint32_t rr = s_runs[r];
              const int which = (32 - __clz((int)(rr - 1))) & 1;  // ceil(log2 rr) parity
              cols[g0 + s_off[r] + idx] = msm[which * kMidBuf + mid_swz(f)];
            }
          }
        }
      }
      __syncthreads();
      q += g;
    }
  }
}

// Centres of a self-query batch in handle order (q[id] = the record's
// point), for the key sorts that need them (range-corner order).
__global__ void self_centres_kernel(const PointRec* __restrict__ rec, uint64_t n,
                                    double* __restrict__ q) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const PointRec pr = rec[i];
    q[3 * (uint64_t)pr.id] = pr.x;
    q[3 * (uint64_t)pr.id + 1] = pr.y;
    q[3 * (uint64_t)pr.id + 2] = pr.z;
  }
}

template <typename K>
cm_status order_typed(const cm_index* ix, const double* q, uint64_t nq, cudaStream_t st,
                      uint32_t* perm, bool range, double r, int kind, int morton_bits = 0,
                      int bz = 0) {
  K* keys = nullptr;
  void* scratch = nullptr;
  CM_CUDA_TRY(dev_alloc_t(&keys, nq, st));
  CM_CUDA_TRY(dev_alloc(&scratch, radix_scratch_bytes<K>(nq), st));
  const unsigned grid = (unsigned)std::min<uint64_t>((nq + 255) / 256, (uint64_t)sm_count() * 16);
  if (morton_bits) {
    query_morton_kernel<K><<<std::max(1u, grid), 256, 0, st>>>(q, nq, ix->g, keys, perm, bz);
    ::cmg::note_launch();
    radix_sort_pairs<K>(keys, perm, nq, morton_bits, scratch, st);
    dev_free(scratch, st);
    dev_free(keys, st);
    return CM_OK;
  }
  if (range)
    query_keys_kernel<K, true><<<std::max(1u, grid), 256, 0, st>>>(q, nq, ix->g, keys, perm, r, kind);
  else
    query_keys_kernel<K, false><<<std::max(1u, grid), 256, 0, st>>>(q, nq, ix->g, keys, perm, r, kind);
  ::cmg::note_launch();
  radix_sort_pairs<K>(keys, perm, nq, ix->key_bits + (range ? 3 : 0), scratch, st);
  dev_free(scratch, st);
  dev_free(keys, st);
  return CM_OK;
}

template <int MODE>
cm_status launch_radius(const cm_index* ix, const double* q, uint64_t nq, int kernel, double r,
                        const uint32_t* perm, const Out& o, cudaStream_t st) {
  const Tables t = ix->tables();
  const size_t smem = (size_t)kQWarps * warp_smem_bytes<MODE>();
  auto run = [&](auto kern) -> cm_status {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kQThreads, smem);
    per_sm = std::max(per_sm, 1);
    const uint64_t need = ((nq + 31) / 32 + kQWarps - 1) / kQWarps;
    const unsigned grid =
        (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(need, (uint64_t)sm_count() * per_sm));
    static const bool no_wide = std::getenv("CMGPU_NO_WIDE") != nullptr;
    Out o2 = o;
    o2.no_wide = no_wide ? 1 : 0;
    kern<<<grid, kQThreads, smem, st>>>(t, q, nq, r, perm, o2); ::cmg::note_launch();
    CM_CUDA_TRY(cudaGetLastError());
    return CM_OK;
  };
  auto pick = [&](auto xq) -> cm_status {
    constexpr bool XQ = decltype(xq)::value;
    switch (ix->opts.flavor) {
      case CM_DENSE:
        return kernel == CM_CUBE       ? run(radius_tile_kernel<CM_DENSE, MODE, 1, XQ>)
               : kernel == CM_CYLINDER ? run(radius_tile_kernel<CM_DENSE, MODE, 2, XQ>)
                                       : run(radius_tile_kernel<CM_DENSE, MODE, 0, XQ>);
      case CM_SPARSE:
        return kernel == CM_CUBE       ? run(radius_tile_kernel<CM_SPARSE, MODE, 1, XQ>)
               : kernel == CM_CYLINDER ? run(radius_tile_kernel<CM_SPARSE, MODE, 2, XQ>)
                                       : run(radius_tile_kernel<CM_SPARSE, MODE, 0, XQ>);
      default:
        return kernel == CM_CUBE       ? run(radius_tile_kernel<CM_MIXED, MODE, 1, XQ>)
               : kernel == CM_CYLINDER ? run(radius_tile_kernel<CM_MIXED, MODE, 2, XQ>)
                                       : run(radius_tile_kernel<CM_MIXED, MODE, 0, XQ>);
    }
  };
  return (o.rq || o.qbox) ? pick(std::true_type{}) : pick(std::false_type{});
}

// Rows longer than a warp buffer (kSortCap), from the one-query-per-warp
// path in COLLECT: written in visit order, i.e. one ascending run per voxel
// (records of a voxel are in handle order), so a row is a few long sorted
// runs (TLS, config 2: up to ~64 voxels per row, thousands of handles each).
// One block per row: find the runs, then merge them pairwise (merge path,
// every thread a fixed slice of the output) — log2(runs) passes instead of
// a bitonic network's log^2(n) stages. Rows that fit go through shared
// memory (two buffers); longer ones ping-pong between their arena row and
// their CSR row, ending in the CSR. More runs than kMergeRunsMax (short
// voxel runs): fixed chunks are bitonic-sorted first and merged the same way.
constexpr int kMergeThreads = 1024;
constexpr uint32_t kMergeSmemElems = 27 * 1024;  // per buffer (two buffers)
constexpr int kMergeRunsMax = 1024;
constexpr uint32_t kMergeChunk = 4096;           // bitonic chunk when runs are short

struct MergeSmem {
  uint32_t buf[2][kMergeSmemElems];
  uint32_t starts[kMergeRunsMax + 2];
  uint32_t swarp[33];
  uint32_t nruns;
};

// One merge pass: runs [starts[r], starts[r + 1]) of `in`, pairs (2p, 2p + 1)
// merged into `out` (same positions); thread t writes outputs
// [t * per, (t + 1) * per). Distinct values: no ties.
__device__ __forceinline__ void merge_pass(const uint32_t* in, uint32_t* out,
                                           const uint32_t* starts, int R, uint32_t n) {
  const uint32_t per = (n + blockDim.x - 1) / blockDim.x;
  uint32_t o = threadIdx.x * per;
  const uint32_t o1 = min(n, o + per);
  if (o >= o1) return;
  // the pair holding output o: the largest p with starts[2p] <= o
  int lo = 0, hi = (R + 1) / 2 - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (starts[2 * mid] <= o) lo = mid; else hi = mid - 1;
  }
  int p = lo;
  while (o < o1) {
    const uint32_t a0 = starts[2 * p];
    const uint32_t a1 = starts[min(2 * p + 1, R)];
    const uint32_t b1 = starts[min(2 * p + 2, R)];
    const uint32_t la = a1 - a0, lb = b1 - a1;
    const uint32_t* A = in + a0;
    const uint32_t* B = in + a1;
    // co-rank of diagonal o - a0
    const uint32_t dg = o - a0;
    uint32_t i0 = dg > lb ? dg - lb : 0u, i1 = min(dg, la);
    while (i0 < i1) {
      const uint32_t mid = (i0 + i1) >> 1;
      if (A[mid] < B[dg - 1 - mid]) i0 = mid + 1; else i1 = mid;
    }
    uint32_t ia = i0, ib = dg - i0;
    const uint32_t oe = min(o1, b1);
    for (; o < oe; ++o) {
      const uint32_t av = ia < la ? A[ia] : 0xffffffffu;
      const uint32_t bv = ib < lb ? B[ib] : 0xffffffffu;
      const bool ta = ib >= lb || (ia < la && av < bv);
      out[o] = ta ? av : bv;
      ia += ta;
      ib += !ta;
    }
    ++p;
  }
}

// starts[] of the ascending runs of a[0..n) (block-wide); returns the run
// count, or kMergeRunsMax + 1 when there are more runs than fit.
__device__ __forceinline__ int find_runs(const uint32_t* a, uint32_t n, MergeSmem& sm) {
  const uint32_t per = (n + blockDim.x - 1) / blockDim.x;
  const uint32_t b = min(n, threadIdx.x * per), e = min(n, b + per);
  uint32_t c = 0;
  for (uint32_t i = b; i < e; ++i) c += (i == 0 || a[i] < a[i - 1]);
  uint32_t tot;
  const uint32_t pos = block_excl_scan<uint32_t>(c, sm.swarp, &tot);
  if (tot <= (uint32_t)kMergeRunsMax) {
    uint32_t w = pos;
    for (uint32_t i = b; i < e; ++i)
      if (i == 0 || a[i] < a[i - 1]) sm.starts[w++] = i;
    if (threadIdx.x == 0) sm.starts[tot] = n;
  }
  __syncthreads();
  return tot <= (uint32_t)kMergeRunsMax ? (int)tot : kMergeRunsMax + 1;
}

// Fixed runs of `chunk` (power of two): each chunk bitonic-sorted through
// shared memory (buf = one smem buffer of >= chunk elements).
__device__ __forceinline__ int chunk_runs(uint32_t* a, uint32_t n, uint32_t chunk, uint32_t* buf,
                                          MergeSmem& sm) {
  for (uint32_t c0 = 0; c0 < n; c0 += chunk) {
    const uint32_t len = min(chunk, n - c0);
    for (uint32_t x = threadIdx.x; x < len; x += blockDim.x) buf[x] = a[c0 + x];
    __syncthreads();
    bitonic_sort(buf, len, threadIdx.x, blockDim.x, [] { __syncthreads(); });
    for (uint32_t x = threadIdx.x; x < len; x += blockDim.x) a[c0 + x] = buf[x];
    __syncthreads();
  }
  const int R = (int)((n + chunk - 1) / chunk);
  for (int r = threadIdx.x; r <= R; r += blockDim.x) sm.starts[r] = r < R ? (uint32_t)r * chunk : n;
  __syncthreads();
  return R;
}

// starts of the merged runs: every other start
__device__ __forceinline__ int halve_runs(MergeSmem& sm, int R, uint32_t n) {
  __syncthreads();
  const int R2 = (R + 1) / 2;
  uint32_t v = 0;
  if ((int)threadIdx.x < R2) v = sm.starts[2 * threadIdx.x];
  __syncthreads();
  if ((int)threadIdx.x < R2) sm.starts[threadIdx.x] = v;
  if (threadIdx.x == 0) sm.starts[R2] = n;
  __syncthreads();
  return R2;
}

__global__ void __launch_bounds__(kMergeThreads) merge_big_rows_kernel(
    uint32_t* __restrict__ arena, const uint64_t* __restrict__ big_off,
    const uint32_t* __restrict__ big_len, const uint32_t* __restrict__ big_q,
    const uint32_t* __restrict__ n_big, const uint64_t* __restrict__ row_ptr,
    uint32_t* __restrict__ cols) {
  extern __shared__ __align__(16) unsigned char msm_raw[];
  MergeSmem& sm = *reinterpret_cast<MergeSmem*>(msm_raw);
  const uint32_t nb = *n_big;
  for (uint32_t bi = blockIdx.x; bi < nb; bi += gridDim.x) {
    const uint32_t n = big_len[bi];
    uint32_t* src = arena + big_off[bi];
    uint32_t* dst = cols + row_ptr[big_q[bi]];
    CM_DCHECK(row_ptr[big_q[bi] + 1] - row_ptr[big_q[bi]] == (uint64_t)n);
    if (n <= kMergeSmemElems) {
      uint32_t* a = sm.buf[0];
      uint32_t* b = sm.buf[1];
      for (uint32_t x = threadIdx.x; x < n; x += blockDim.x) a[x] = src[x];
      __syncthreads();
      int R = find_runs(a, n, sm);
      if (R > kMergeRunsMax) {
        R = chunk_runs(a, n, kMergeChunk, b, sm);
      }
      while (R > 1) {
        merge_pass(a, b, sm.starts, R, n);
        R = halve_runs(sm, R, n);
        uint32_t* t = a;
        a = b;
        b = t;
      }
      for (uint32_t x = threadIdx.x; x < n; x += blockDim.x) dst[x] = a[x];
    } else {
      int R = find_runs(src, n, sm);
      if (R > kMergeRunsMax) {
        // chunk size: a power of two with at most kMergeRunsMax chunks
        uint32_t ch = kMergeChunk;
        while ((n + ch - 1) / ch > (uint32_t)kMergeRunsMax && ch < 16384u) ch <<= 1;
        R = chunk_runs(src, n, ch, sm.buf[0], sm);
      }
      // ping-pong src <-> dst; an even number of passes ends in src
      uint32_t* a = src;
      uint32_t* b = dst;
      while (R > 1) {
        merge_pass(a, b, sm.starts, R, n);
        R = halve_runs(sm, R, n);
        uint32_t* t = a;
        a = b;
        b = t;
      }
      if (a != dst)
        for (uint32_t x = threadIdx.x; x < n; x += blockDim.x) dst[x] = a[x];
    }
    __syncthreads();
  }
}

}  // namespace

uint32_t long_row_min() { return (uint32_t)kSortCap + 1u; }

namespace {

cm_status merge_big_rows_impl(uint32_t* arena, const uint64_t* big_off, const uint32_t* big_len,
                         const uint32_t* big_q, const uint32_t* n_big, const uint64_t* row_ptr,
                         uint32_t* cols, cudaStream_t st) {
  const int smem = (int)sizeof(MergeSmem);
  cudaFuncSetAttribute(merge_big_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  merge_big_rows_kernel<<<sm_count(), kMergeThreads, smem, st>>>(arena, big_off, big_len, big_q,
                                                                 n_big, row_ptr, cols);
  ::cmg::note_launch();
  CM_CUDA_TRY(cudaGetLastError());
  return CM_OK;
}

}  // namespace

cm_status merge_big_rows(const MergeList& ml, uint32_t* arena, const uint64_t* row_ptr,
                         uint32_t* cols, cudaStream_t st) {
  return merge_big_rows_impl(arena, ml.off, ml.len, ml.q, ml.n, row_ptr, cols, st);
}

namespace {

cm_status sort_big_rows(uint32_t* rows, const Out& o, cudaStream_t st) {
  const int smem = kBigSmemCap * 4;
  cudaFuncSetAttribute(big_row_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  big_row_sort_kernel<<<sm_count(), 1024, smem, st>>>(rows, o.big_off, o.big_len, o.n_big); ::cmg::note_launch();
  CM_CUDA_TRY(cudaGetLastError());
  return CM_OK;
}

struct BigRows {
  uint64_t* off = nullptr;
  uint32_t* len = nullptr;
  uint32_t* n = nullptr;
  cudaStream_t st = nullptr;
  cm_status init(uint64_t nq, cudaStream_t s) {
    st = s;
    CM_CUDA_TRY(dev_alloc_t(&off, nq, s));
    CM_CUDA_TRY(dev_alloc_t(&len, nq, s));
    CM_CUDA_TRY(dev_alloc_t(&n, 1, s));
    CM_CUDA_TRY(cudaMemsetAsync(n, 0, 4, s));
    return CM_OK;
  }
  ~BigRows() {
    dev_free(off, st);
    dev_free(len, st);
    dev_free(n, st);
  }
};

}  // namespace

void query_stats(uint64_t* out, int reset) {
  unsigned long long h[8];
  cudaMemcpyFromSymbol(h, g_qstats, sizeof(h));
  for (int i = 0; i < 8; ++i) out[i] = h[i];
  if (reset) {
    const unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_qstats, z, sizeof(z));
  }
}

static int bit_width_u64(uint64_t v) {
  int b = 0;
  while (v) ++b, v >>= 1;
  return b;
}

cm_status order_queries(const cm_index* ix, const double* q, uint64_t nq, cudaStream_t st,
                        QueryOrder* out, double r, int kind, bool morton) {
  out->nq = nq;
  out->st = st;
  out->q = q;
  if (nq == 0) return CM_OK;
  const DevGrid& g = ix->g;
  auto fits = [&](double f) {  // f = 2: every clamped range spans at most 2 cells per axis
    return r >= 0.0 && f * r <= g.sx && f * r <= g.sy &&
           (!g.mode3d || kind == CM_CYLINDER || f * r <= g.sz);
  };
  // (2-bit extents for r <= cell, ranges of up to 3 cells, measured no gain at r = 1)
  const bool range = fits(2.0);
  if (q == nullptr) {
    // Self queries (cm_radius_search_self: every indexed point a centre, row
    // q = point q): the records' cell order IS the order the centre-key sort
    // would produce, so the kernels read centres straight from the records
    // (out->q stays null, no permutation). Range-corner order differs from
    // cell order, so for those radii the centres are materialised in handle
    // order and sorted like any batch.
    if (!range) return CM_OK;
    if (nq != ix->n) return CM_INVALID_ARGUMENT;
    CM_CUDA_TRY(dev_alloc_t(&out->owned_q, nq * 3, st));
    const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((nq + 255) / 256, (uint64_t)sm_count() * 16));
    self_centres_kernel<<<grid, 256, 0, st>>>(ix->rec, nq, out->owned_q); ::cmg::note_launch();
    CM_CUDA_TRY(cudaGetLastError());
    q = out->owned_q;
  }
  out->q = q;
  CM_CUDA_TRY(dev_alloc_t(&out->perm, nq, st));
  if (morton && q) {
    const int bxy = bit_width_u64(std::max(g.nx, g.ny) - 1);
    const int bz = g.mode3d ? bit_width_u64(g.nz - 1) : 0;
    const int mb = 2 * bxy + bz;
    if (bxy <= 21 && mb <= 64) {
      return mb <= 32 ? order_typed<uint32_t>(ix, q, nq, st, out->perm, false, r, kind, std::max(1, mb), bz)
                      : order_typed<uint64_t>(ix, q, nq, st, out->perm, false, r, kind, mb, bz);
    }
  }
  const int bits = ix->key_bits + (range ? 3 : 0);
  return bits <= 32 ? order_typed<uint32_t>(ix, q, nq, st, out->perm, range, r, kind)
                    : order_typed<uint64_t>(ix, q, nq, st, out->perm, range, r, kind);
}

// Radii whose clamped ranges span more columns than a compact 32-column
// tile hull can hold: rows come from wide tiles (count + fill + row sort).
bool radius_is_wide(const cm_index* ix, double r) {
  const double cx = std::floor(2.0 * r / ix->g.sx) + 2.0;
  const double cy = std::floor(2.0 * r / ix->g.sy) + 2.0;
  return cx * cy > 20.0;
}

cm_status radius_count_dev(const cm_index* ix, const double* q, uint64_t nq, int kernel, double r,
                           const uint32_t* perm, uint32_t* counts, uint64_t* tested,
                           cudaStream_t st, const double* rq, const double* qbox) {
  if (nq == 0) return CM_OK;
  Out o{};
  o.counts = counts;
  o.tested = tested;
  o.rq = rq;
  o.qbox = qbox;
  return launch_radius<MODE_COUNT>(ix, q, nq, kernel, r, perm, o, st);
}

cm_status radius_digest_dev(const cm_index* ix, const double* q, uint64_t nq, int kernel, double r,
                            const uint32_t* perm, uint32_t* counts, uint64_t* digests,
                            cudaStream_t st, const double* rq, const double* qbox) {
  if (nq == 0) return CM_OK;
  Out o{};
  o.counts = counts;
  o.digests = digests;
  o.rq = rq;
  o.qbox = qbox;
  return launch_radius<MODE_DIGEST>(ix, q, nq, kernel, r, perm, o, st);
}

// Rows of 513..1024 handles, from the count pass: out[0] = how many,
// out[1] = their total length (the row-sort plan of a wide FILL).
__global__ void row_class_kernel(const uint32_t* __restrict__ counts, uint64_t nq,
                                 unsigned long long* __restrict__ out) {
  unsigned long long a = 0, b = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nq;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t c = __ldg(counts + i);
    const bool in = c > 512u && c <= 1024u;
    a += in;
    b += in ? c : 0u;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (a) atomicAdd(out, a);
    if (b) atomicAdd(out + 1, b);
  }
}

cm_status row_class_counts_dev(const uint32_t* counts, uint64_t nq, unsigned long long* out,
                               cudaStream_t st) {
  CM_CUDA_TRY(cudaMemsetAsync(out, 0, 16, st));
  if (nq == 0) return CM_OK;
  const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((nq + 255) / 256, (uint64_t)sm_count() * 8));
  row_class_kernel<<<grid, 256, 0, st>>>(counts, nq, out); ::cmg::note_launch();
  CM_CUDA_TRY(cudaGetLastError());
  return CM_OK;
}

cm_status radius_fill_dev(const cm_index* ix, const double* q, uint64_t nq, int kernel, double r,
                          const uint32_t* perm, const uint64_t* row_ptr, uint32_t* cols,
                          cudaStream_t st, cudaEvent_t after_fill, uint32_t mid_min,
                          const double* rq, const double* qbox) {
  if (nq == 0) return CM_OK;
  if (mid_min == 0) mid_min = (uint32_t)kMidMin;
  BigRows big;
  cm_status s = big.init(nq, st);
  if (s != CM_OK) return s;
  Out o{};
  o.row_ptr = row_ptr;
  o.cols = cols;
  o.big_off = big.off;
  o.big_len = big.len;
  o.n_big = big.n;
  o.wide_fill = (radius_is_wide(ix, r) || rq || qbox) ? 1 : 0;
  o.rq = rq;
  o.qbox = qbox;
  s = launch_radius<MODE_FILL>(ix, q, nq, kernel, r, perm, o, st);
  if (after_fill) cudaEventRecord(after_fill, st);
  if (s != CM_OK) return s;
  if (!o.wide_fill) return sort_big_rows(cols, o, st);
  // wide tiles left rows unsorted: sort every row in place
  BigRows big2;
  s = big2.init(nq, st);
  if (s != CM_OK) return s;
  const uint64_t groups = (nq + 31) / 32;
  const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((groups + 3) / 4, (uint64_t)sm_count() * 8));
  const int smem = 4 * kGatherWarpWords * 4;
  cudaFuncSetAttribute(gather_rows_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  gather_rows_kernel<true><<<grid, 128, smem, st>>>(cols, row_ptr, nullptr, row_ptr, cols, nq); ::cmg::note_launch();
  CM_CUDA_TRY(cudaGetLastError());
  {
    const unsigned bgrid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((groups + 3) / 4, (uint64_t)sm_count() * 16));
    sort_blocked_rows_kernel<4><<<bgrid, 128, 0, st>>>(cols, row_ptr, nq, kGatherRow); ::cmg::note_launch();
    if (kMidMin > 128) {
      sort_blocked_rows_kernel<8><<<bgrid, 128, 0, st>>>(cols, row_ptr, nq, 128); ::cmg::note_launch();
    }
    if (kMidMin > 256) {
      sort_blocked_rows_kernel<16><<<bgrid, 128, 0, st>>>(cols, row_ptr, nq, 256); ::cmg::note_launch();
    }
    // 513..1024: head 512 + tail + merge (measured: r = 5 fill + sort 44.4 ->
    // 42.0 ms; for the shorter classes the padded network stays faster)
    const int ssmem = 4 * kSplitWarpWords * 4;
    cudaFuncSetAttribute(sort_split_rows_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, ssmem);
    if (mid_min > 512) {
      sort_split_rows_kernel<16><<<bgrid, 128, ssmem, st>>>(cols, row_ptr, nq); ::cmg::note_launch();
    }

    CM_CUDA_TRY(cudaGetLastError());
  }
  {
    const int msmem = 2 * kMidBuf * 4;
    cudaFuncSetAttribute(sort_mid_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, msmem);
    const uint64_t tasks = (nq + 1023) / 1024;
    const unsigned mgrid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(tasks, (uint64_t)sm_count() * 3));
    sort_mid_rows_kernel<<<mgrid, kMidThreads, msmem, st>>>(cols, row_ptr, nq, big2.off, big2.len,
                                                            big2.n, mid_min); ::cmg::note_launch();
  }
  CM_CUDA_TRY(cudaGetLastError());
  Out o2{};
  o2.big_off = big2.off;
  o2.big_len = big2.len;
  o2.n_big = big2.n;
  return sort_big_rows(cols, o2, st);
}

cm_status radius_collect_dev(const cm_index* ix, const double* q, uint64_t nq, int kernel,
                             double r, const uint32_t* perm, uint32_t* temp, uint64_t cap,
                             uint64_t* toff, uint32_t* scnt, uint32_t* counts,
                             unsigned long long* cursor, cudaStream_t st,
                             cudaEvent_t after_collect, const double* rq, const double* qbox,
                             const MergeList* ml) {
  // the caller reads the cursor and the merge list even for nq = 0
  CM_CUDA_TRY(cudaMemsetAsync(cursor, 0, 16, st));
  if (ml) CM_CUDA_TRY(cudaMemsetAsync(ml->n, 0, 4, st));
  if (nq == 0) return CM_OK;
  BigRows big;
  cm_status s = ml ? CM_OK : big.init(nq, st);
  if (s != CM_OK) return s;
  Out o{};
  o.counts = counts;
  o.temp = temp;
  o.cap = cap;
  o.toff = toff;
  o.scnt = scnt;
  o.cursor = cursor;
  o.nnz = cursor + 1;
  o.big_off = ml ? ml->off : big.off;
  o.big_len = ml ? ml->len : big.len;
  o.big_q = ml ? ml->q : nullptr;
  o.n_big = ml ? ml->n : big.n;
  o.rq = rq;
  o.qbox = qbox;
  s = launch_radius<MODE_COLLECT>(ix, q, nq, kernel, r, perm, o, st);
  if (after_collect) cudaEventRecord(after_collect, st);
  // with a merge list the long rows stay in visit order (sorted runs) for
  // merge_big_rows after the scan; otherwise they are sorted here in place
  if (s == CM_OK && !ml) s = sort_big_rows(temp, o, st);
  return s;
}

cm_status gather_rows_dev(const uint32_t* temp, const uint64_t* toff, const uint32_t* counts,
                          const uint64_t* row_ptr, const uint32_t* perm, uint32_t* cols,
                          uint64_t nq, cudaStream_t st, uint32_t skip_above) {
  if (nq == 0) return CM_OK;
  const uint64_t groups = (nq + 31) / 32;
  const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((groups + 3) / 4, (uint64_t)sm_count() * 8));
  const int smem = 4 * kGatherWarpWords * 4;
  (void)perm;
  cudaFuncSetAttribute(gather_rows_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  gather_rows_kernel<false><<<grid, 128, smem, st>>>(temp, toff, counts, row_ptr, cols, nq,
                                                     skip_above);
  ::cmg::note_launch();
  CM_CUDA_TRY(cudaGetLastError());
  return CM_OK;
}

namespace {
// weighted_density's binning (analysis.cpp:67-70): local = count / pi,
// bin = min(255, (u64)local); per-block shared histograms.
__global__ void density_hist_kernel(const uint32_t* __restrict__ counts, uint64_t n,
                                    unsigned long long* __restrict__ bins) {
  __shared__ uint32_t h[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
  __syncthreads();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const double local = __ddiv_rn((double)counts[i], 3.141592653589793);
    const uint64_t b = (uint64_t)local;
    atomicAdd(&h[b < 255 ? b : 255], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x)
    if (h[i]) atomicAdd(bins + i, (unsigned long long)h[i]);
}

__global__ void gather_points_kernel(const double* __restrict__ xyz,
                                     const uint64_t* __restrict__ idx, uint64_t n,
                                     double* __restrict__ out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t h = idx[i];
    out[3 * i] = xyz[3 * h];
    out[3 * i + 1] = xyz[3 * h + 1];
    out[3 * i + 2] = xyz[3 * h + 2];
  }
}
}  // namespace

cm_status density_histogram_dev(const uint32_t* counts, uint64_t n, unsigned long long* bins,
                                cudaStream_t st) {
  CM_CUDA_TRY(cudaMemsetAsync(bins, 0, 256 * 8, st));
  if (n) {
    const unsigned grid = (unsigned)std::max<uint64_t>(
        1, std::min<uint64_t>((n + 255) / 256, (uint64_t)sm_count() * 8));
    density_hist_kernel<<<grid, 256, 0, st>>>(counts, n, bins); ::cmg::note_launch();
  }
  CM_CUDA_TRY(cudaGetLastError());
  return CM_OK;
}

cm_status gather_points_dev(const double* xyz, const uint64_t* idx, uint64_t n, double* out,
                            cudaStream_t st) {
  if (!n) return CM_OK;
  const unsigned grid =
      (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, (uint64_t)sm_count() * 8));
  gather_points_kernel<<<grid, 256, 0, st>>>(xyz, idx, n, out); ::cmg::note_launch();
  CM_CUDA_TRY(cudaGetLastError());
  return CM_OK;
}

cm_status counts_to_row_ptr(const uint32_t* counts, uint64_t nq, uint64_t* row_ptr,
                            cudaStream_t st) {
  uint64_t* part = nullptr;
  CM_CUDA_TRY(dev_alloc_t(&part, scan_part_elems(nq), st));
  exclusive_scan<uint32_t, uint64_t>(counts, nq, row_ptr, part, 1, st);
  dev_free(part, st);
  CM_CUDA_TRY(cudaGetLastError());
  return CM_OK;
}

}  // namespace cmg
