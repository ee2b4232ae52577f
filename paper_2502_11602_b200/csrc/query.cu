// Batched fixed-radius queries (sphere / cube) on sm_100a.
// Replaces kernel_search<Kernel> (search.hpp:102-127) for a batch of centres.
//
// Pipeline: query cell keys -> radix sort (spatial order, so neighbouring
// warps touch the same candidate records in L1/L2) -> warp-per-query count
// (K5) -> exclusive scan (K6) -> warp-per-query fill + in-warp bitonic sort
// of each row (K7). Rows too long for the per-warp buffer are written
// unsorted and sorted afterwards by a persistent block-per-row kernel.
//
// Candidate enumeration is exactly the reference's: every point of every
// voxel of clamped_range(c +- r) (grid.cpp:90-114). The points of one
// (i, j) column inside [k0, k1] are one contiguous span of the cell-sorted
// records, so a query is ncol spans; the warp flattens them and tests 32
// candidates per step with the reference's predicate arithmetic.
#include <algorithm>

#include "index.cuh"
#include "sort_scan.cuh"

namespace cmg {

namespace {

constexpr int kQThreads = 128;
constexpr int kQWarps = kQThreads / 32;
constexpr int kTileCap = 512;                  // hull points per warp (fill pass)
constexpr int kFillWarpBytes = kTileCap * 12;  // u64 keys + u32 positions
constexpr int kRowCap = kFillWarpBytes / 4;    // fallback per-warp row buffer (u32)
constexpr int kBigSmemCap = 32768;  // block sort in shared memory (128 KB)

enum { MODE_COUNT = 0, MODE_FILL = 1, MODE_DIGEST = 2 };

// Tile statistics (cm_debug_query_stats): [0] tiles, [1] fallback tiles,
// [2] staged points (tile mode), [3] in-range candidates (tile mode).
__device__ unsigned long long g_qstats[4];

template <typename K>
__global__ void query_keys_kernel(const double* __restrict__ q, uint64_t nq, DevGrid g,
                                  K* __restrict__ keys, uint32_t* __restrict__ vals) {
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < nq;
       p += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = axis_index(q[3 * p], g.ox, g.sx, g.nx);
    const uint64_t j = axis_index(q[3 * p + 1], g.oy, g.sy, g.ny);
    const uint64_t k = g.mode3d ? axis_index(q[3 * p + 2], g.oz, g.sz, g.nz) : 0;
    keys[p] = (K)(i * (g.ny * g.nz) + j * g.nz + k);
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
template <int FLAVOR, int MODE>
__device__ __forceinline__ void query_warp(const Tables& t, uint32_t qi, double cx, double cy,
                                           double cz, double r, int cube, int lane, uint32_t lt,
                                           uint32_t* counts, uint64_t* tested, uint64_t* digests,
                                           const uint64_t* row_ptr, uint32_t* cols,
                                           uint32_t* big_rows, uint32_t* n_big, uint32_t* wbuf) {
  Range R;
  const bool ok = clamped_range(t.g, cx, cy, cz, r, &R);
  Predicate P;
  P.init(cx, cy, cz, r, cube);
  uint32_t cnt = 0;
  uint64_t ntested = 0, dig = 0;
  uint64_t rowb = 0;
  bool direct = false;
  if (MODE == MODE_FILL) {
    rowb = __ldg(row_ptr + qi);
    direct = (__ldg(row_ptr + qi + 1) - rowb) > (uint64_t)kRowCap;
  }
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
        uint32_t id = 0;
        if (tt < total) {
          const PointRec pr = load_rec(t.rec + bL + (tt - xL));
          hit = P(pr.x, pr.y, pr.z);
          id = pr.id;
        }
        const uint32_t m = __ballot_sync(0xffffffffu, hit);
        if (MODE == MODE_DIGEST && hit) dig += mix64(id);
        if (MODE == MODE_FILL && hit) {
          const uint32_t off = cnt + __popc(m & lt);
          if (direct) cols[rowb + off] = id;
          else wbuf[off] = id;
        }
        cnt += __popc(m);
      }
    }
  }
  if (MODE == MODE_COUNT) {
    if (lane == 0) {
      if (counts) counts[qi] = cnt;
      if (tested) tested[qi] = ntested;
    }
  } else if (MODE == MODE_DIGEST) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dig += __shfl_xor_sync(0xffffffffu, dig, o);
    if (lane == 0) {
      counts[qi] = cnt;
      digests[qi] = dig;
    }
  } else {
    if (direct) {
      if (lane == 0) big_rows[atomicAdd(n_big, 1u)] = qi;
    } else if (cnt <= 32) {
      __syncwarp();
      uint32_t v = lane < (int)cnt ? wbuf[lane] : 0xffffffffu;
      v = warp_sort32(v, lane);
      if (lane < (int)cnt) cols[rowb + lane] = v;
    } else {
      __syncwarp();
      bitonic_sort(wbuf, cnt, lane, 32, [] { __syncwarp(); });
      for (uint32_t x = lane; x < cnt; x += 32) cols[rowb + x] = wbuf[x];
    }
  }
  __syncwarp();
}

// Ascending bitonic sort of a[0..n) (u64) by one warp; P = pow2 >= n,
// indices >= n act as +inf. Iterates compare pairs directly.
__device__ __forceinline__ void warp_bitonic_u64(uint64_t* a, uint32_t n, int lane) {
  uint32_t P = 1, lg = 0;
  while (P < n) P <<= 1, ++lg;
  const uint32_t half = P >> 1;
  for (uint32_t lk = 1; lk <= lg; ++lk) {
    const uint32_t k = 1u << lk;
    // flip step: i in the lower half of its k-block, partner i ^ (k - 1)
    for (uint32_t tq = lane; tq < half; tq += 32) {
      const uint32_t i = ((tq >> (lk - 1)) << lk) | (tq & ((k >> 1) - 1));
      const uint32_t p = i ^ (k - 1);
      if (p < n) {
        const uint64_t x = a[i], y = a[p];
        if (x > y) {
          a[i] = y;
          a[p] = x;
        }
      }
    }
    __syncwarp();
    for (int lj = (int)lk - 2; lj >= 0; --lj) {
      const uint32_t j = 1u << lj;
      for (uint32_t tq = lane; tq < half; tq += 32) {
        const uint32_t i = ((tq >> lj) << (lj + 1)) | (tq & (j - 1));
        const uint32_t p = i + j;
        if (p < n) {
          const uint64_t x = a[i], y = a[p];
          if (x > y) {
            a[i] = y;
            a[p] = x;
          }
        }
      }
      __syncwarp();
    }
  }
}

__device__ __forceinline__ uint32_t warp_min_u32(uint32_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ uint32_t warp_max_u32(uint32_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

template <int CUBE>
__device__ __forceinline__ bool pred(const Predicate& P, double x, double y, double z) {
  if (CUBE)
    return (x >= P.lx) & (x <= P.hx) & (y >= P.ly) & (y <= P.hy) & (z >= P.lz) & (z <= P.hz);
  return sqdist(x, y, z, P.cx, P.cy, P.cz) <= P.rr;
}

// Warp-uniform record read: every lane loads the same 32 bytes (one L1
// wavefront each, broadcast).
__device__ __forceinline__ void load_uniform(const PointRec* p, double& x, double& y, double& z,
                                             uint32_t& id, uint32_t& k) {
  const double2 a = __ldg(reinterpret_cast<const double2*>(p));
  const double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
  x = a.x;
  y = a.y;
  z = b.x;
  const uint2 t = *reinterpret_cast<const uint2*>(&b.y);
  id = t.x;
  k = t.y;
}

// Query-tile kernel. A warp takes 32 consecutive (cell-sorted) queries, one
// per lane. When their clamped ranges have a compact hull (<= 32 columns,
// <= kTileCap points), the warp walks the hull's points once, warp-uniformly
// (every lane reads the same record: an L1 broadcast), and each lane tests
// each point against its own query: a point counts for lane q only if its
// voxel lies in q's own clamped_range (the reference's exact candidate set,
// search.hpp:110-122) and q's predicate holds. The fill pass first sorts the
// hull's (handle, slot) keys in shared memory, so each lane's hits come out
// ascending and go straight to its CSR row. Tiles that are not compact fall
// back to query_warp for each of their queries.
template <int FLAVOR, int MODE, int CUBE>
__global__ void __launch_bounds__(kQThreads, 4) radius_tile_kernel(
    const Tables t, const double* __restrict__ q, uint64_t nq, double r,
    const uint32_t* __restrict__ perm, uint32_t* __restrict__ counts,
    uint64_t* __restrict__ tested, uint64_t* __restrict__ digests,
    const uint64_t* __restrict__ row_ptr, uint32_t* __restrict__ cols,
    uint32_t* __restrict__ big_rows, uint32_t* __restrict__ n_big) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  unsigned char* wbase = smraw + (size_t)wib * kFillWarpBytes;
  uint64_t* skey = reinterpret_cast<uint64_t*>(wbase);                  // kTileCap
  uint32_t* spos = reinterpret_cast<uint32_t*>(wbase + kTileCap * 8);   // kTileCap
  uint32_t* wbuf = reinterpret_cast<uint32_t*>(wbase);                  // fallback rows
  const uint32_t lt = lanemask_lt();
  const uint64_t ntiles = (nq + 31) / 32;
  const uint64_t W = (uint64_t)gridDim.x * kQWarps;
  const bool small_grid = t.g.nx < (1ull << 31) && t.g.ny < (1ull << 31) && t.g.nz < (1ull << 31);
  const PointRec* __restrict__ rec = t.rec;

  for (uint64_t tile = (uint64_t)blockIdx.x * kQWarps + wib; tile < ntiles; tile += W) {
    const uint64_t s = tile * 32 + lane;
    const bool active = s < nq;
    const uint32_t qi = active ? __ldg(perm + s) : 0u;
    double cx = 0.0, cy = 0.0, cz = 0.0;
    if (active) {
      cx = __ldg(q + 3 * (uint64_t)qi);
      cy = __ldg(q + 3 * (uint64_t)qi + 1);
      cz = __ldg(q + 3 * (uint64_t)qi + 2);
    }
    Range R{};
    const bool ok = active && clamped_range(t.g, cx, cy, cz, r, &R);
    const uint32_t okmask = __ballot_sync(0xffffffffu, ok);
    bool use_tile = small_grid && okmask != 0;
    uint32_t I0 = 0, J0 = 0, nj = 0, ncol = 0, total = 0;
    uint32_t b = 0, e = 0, incl = 0, excl = 0;
    if (use_tile) {
      I0 = warp_min_u32(ok ? (uint32_t)R.i0 : 0xffffffffu);
      const uint32_t I1 = warp_max_u32(ok ? (uint32_t)R.i1 : 0u);
      J0 = warp_min_u32(ok ? (uint32_t)R.j0 : 0xffffffffu);
      const uint32_t J1 = warp_max_u32(ok ? (uint32_t)R.j1 : 0u);
      const uint32_t K0 = warp_min_u32(ok ? (uint32_t)R.k0 : 0xffffffffu);
      const uint32_t K1 = warp_max_u32(ok ? (uint32_t)R.k1 : 0u);
      nj = J1 - J0 + 1;
      const uint64_t nc = (uint64_t)(I1 - I0 + 1) * nj;
      use_tile = nc <= 32;
      if (use_tile) {
        ncol = (uint32_t)nc;
        if ((uint32_t)lane < ncol)
          column_span<FLAVOR>(t, I0 + lane / nj, J0 + lane % nj, K0, K1, &b, &e);
        const uint32_t len = e - b;
        incl = warp_incl_scan(len);
        excl = incl - len;
        total = __shfl_sync(0xffffffffu, incl, 31);
        use_tile = MODE != MODE_FILL || total <= (uint32_t)kTileCap;
        if (lane == 0) {
          atomicAdd(&g_qstats[0], 1ull);
          if (use_tile) atomicAdd(&g_qstats[2], (unsigned long long)total);
          else atomicAdd(&g_qstats[1], 1ull);
        }
      } else if (lane == 0) {
        atomicAdd(&g_qstats[0], 1ull);
        atomicAdd(&g_qstats[1], 1ull);
      }
    }
    if (!use_tile) {
      const uint32_t am = __ballot_sync(0xffffffffu, active);
      for (int l = 0; l < 32; ++l) {
        if (!((am >> l) & 1u)) continue;
        const uint32_t ql = __shfl_sync(0xffffffffu, qi, l);
        const double xl = __shfl_sync(0xffffffffu, cx, l);
        const double yl = __shfl_sync(0xffffffffu, cy, l);
        const double zl = __shfl_sync(0xffffffffu, cz, l);
        query_warp<FLAVOR, MODE>(t, ql, xl, yl, zl, r, CUBE, lane, lt, counts, tested, digests,
                                 row_ptr, cols, big_rows, n_big, wbuf);
      }
      continue;
    }
    // this lane's columns within the hull, and its k window
    uint32_t colmask = 0;
    if (ok) {
      const uint64_t rowbits = ((1ull << ((uint32_t)(R.j1 - R.j0) + 1)) - 1ull) << ((uint32_t)R.j0 - J0);
      for (uint32_t ci = (uint32_t)R.i0 - I0; ci <= (uint32_t)R.i1 - I0; ++ci)
        colmask |= (uint32_t)(rowbits << (ci * nj));
    }
    const uint32_t kk0 = ok ? (uint32_t)R.k0 : 1u;
    const uint32_t kspan = ok ? (uint32_t)(R.k1 - R.k0) : 0u;
    Predicate P;
    P.init(cx, cy, cz, r, CUBE);
    uint32_t cnt = 0, ntest = 0;
    uint64_t dig = 0;
    if (MODE != MODE_FILL) {
      // column by column, in stored order
      for (uint32_t c = 0; c < ncol; ++c) {
        const uint32_t cb = __shfl_sync(0xffffffffu, b, c);
        const uint32_t ce = __shfl_sync(0xffffffffu, e, c);
        const bool need = (colmask >> c) & 1u;
        if (__ballot_sync(0xffffffffu, need) == 0) continue;
        uint32_t p = cb;
        for (; p + 4 <= ce; p += 4) {
          double x[4], y[4], z[4];
          uint32_t id[4], kz[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) load_uniform(rec + p + u, x[u], y[u], z[u], id[u], kz[u]);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const bool in = need & (kz[u] - kk0 <= kspan);
            const bool hit = in & pred<CUBE>(P, x[u], y[u], z[u]);
            if (MODE == MODE_DIGEST && hit) dig += mix64(id[u]);
            cnt += hit;
            ntest += in;
          }
        }
        for (; p < ce; ++p) {
          double x, y, z;
          uint32_t id, kz;
          load_uniform(rec + p, x, y, z, id, kz);
          const bool in = need & (kz - kk0 <= kspan);
          const bool hit = in & pred<CUBE>(P, x, y, z);
          if (MODE == MODE_DIGEST && hit) dig += mix64(id);
          cnt += hit;
          ntest += in;
        }
      }
    } else {
      // keys (handle << 32 | column << 16 | slot) and record positions
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
        if (tt < total) {
          const uint32_t pos = bL + (tt - xL);
          const uint32_t id = __ldg(reinterpret_cast<const uint32_t*>(rec + pos) + 6);
          skey[tt] = ((uint64_t)id << 32) | ((uint32_t)L << 16) | tt;
          spos[tt] = pos;
        }
      }
      __syncwarp();
      warp_bitonic_u64(skey, total, lane);
      const uint64_t rowb = active ? __ldg(row_ptr + qi) : 0;
      uint32_t u = 0;
      for (; u + 4 <= total; u += 4) {
        double x[4], y[4], z[4];
        uint32_t id[4], kz[4], col[4];
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const uint64_t key = skey[u + v];
          col[v] = ((uint32_t)key >> 16) & 0xffffu;
          load_uniform(rec + spos[(uint32_t)key & 0xffffu], x[v], y[v], z[v], id[v], kz[v]);
        }
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const bool in = ((colmask >> col[v]) & 1u) & (kz[v] - kk0 <= kspan);
          const bool hit = in & pred<CUBE>(P, x[v], y[v], z[v]);
          if (hit) cols[rowb + cnt] = id[v];
          cnt += hit;
        }
      }
      for (; u < total; ++u) {
        const uint64_t key = skey[u];
        const uint32_t cl = ((uint32_t)key >> 16) & 0xffffu;
        double x, y, z;
        uint32_t id, kz;
        load_uniform(rec + spos[(uint32_t)key & 0xffffu], x, y, z, id, kz);
        const bool in = ((colmask >> cl) & 1u) & (kz - kk0 <= kspan);
        const bool hit = in & pred<CUBE>(P, x, y, z);
        if (hit) cols[rowb + cnt] = id;
        cnt += hit;
      }
    }
    if (MODE == MODE_COUNT) {
      uint32_t sum = ntest;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      if (lane == 0) atomicAdd(&g_qstats[3], (unsigned long long)sum);
    }
    if (active) {
      if (MODE == MODE_COUNT) {
        if (counts) counts[qi] = cnt;
        if (tested) tested[qi] = ntest;
      } else if (MODE == MODE_DIGEST) {
        counts[qi] = cnt;
        digests[qi] = dig;
      }
    }
    __syncwarp();
  }
}

// Rows longer than the per-warp buffer: one block per row (persistent).
__global__ void __launch_bounds__(1024) big_row_sort_kernel(const uint64_t* __restrict__ row_ptr,
                                                            uint32_t* __restrict__ cols,
                                                            const uint32_t* __restrict__ big_rows,
                                                            const uint32_t* __restrict__ n_big) {
  extern __shared__ uint32_t sm[];
  const uint32_t nb = *n_big;
  for (uint32_t b = blockIdx.x; b < nb; b += gridDim.x) {
    const uint32_t qi = big_rows[b];
    const uint64_t beg = row_ptr[qi];
    const uint32_t len = (uint32_t)(row_ptr[qi + 1] - beg);
    uint32_t* row = cols + beg;
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

template <typename K>
cm_status order_typed(const cm_index* ix, const double* q, uint64_t nq, cudaStream_t st,
                      uint32_t* perm) {
  K* keys = nullptr;
  void* scratch = nullptr;
  CM_CUDA_TRY(dev_alloc_t(&keys, nq, st));
  CM_CUDA_TRY(dev_alloc(&scratch, radix_scratch_bytes<K>(nq), st));
  const unsigned grid = (unsigned)std::min<uint64_t>((nq + 255) / 256, (uint64_t)sm_count() * 16);
  query_keys_kernel<K><<<std::max(1u, grid), 256, 0, st>>>(q, nq, ix->g, keys, perm); ::cmg::note_launch();
  radix_sort_pairs<K>(keys, perm, nq, ix->key_bits, scratch, st);
  dev_free(scratch, st);
  dev_free(keys, st);
  return CM_OK;
}

template <int MODE>
cm_status launch_radius(const cm_index* ix, const double* q, uint64_t nq, int kernel, double r,
                        const uint32_t* perm, uint32_t* counts, uint64_t* tested,
                        uint64_t* digests, const uint64_t* row_ptr, uint32_t* cols,
                        uint32_t* big_rows, uint32_t* n_big, cudaStream_t st) {
  const Tables t = ix->tables();
  const size_t smem = MODE == MODE_FILL ? (size_t)kQWarps * kFillWarpBytes : 0;
  auto run = [&](auto kern) -> cm_status {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kQThreads, smem);
    per_sm = std::max(per_sm, 1);
    const uint64_t need = ((nq + 31) / 32 + kQWarps - 1) / kQWarps;
    const unsigned grid =
        (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(need, (uint64_t)sm_count() * per_sm));
    kern<<<grid, kQThreads, smem, st>>>(t, q, nq, r, perm, counts, tested, digests, row_ptr, cols,
                                        big_rows, n_big); ::cmg::note_launch();
    CM_CUDA_TRY(cudaGetLastError());
    return CM_OK;
  };
  switch (ix->opts.flavor) {
    case CM_DENSE:
      return kernel == CM_CUBE ? run(radius_tile_kernel<CM_DENSE, MODE, 1>)
                               : run(radius_tile_kernel<CM_DENSE, MODE, 0>);
    case CM_SPARSE:
      return kernel == CM_CUBE ? run(radius_tile_kernel<CM_SPARSE, MODE, 1>)
                               : run(radius_tile_kernel<CM_SPARSE, MODE, 0>);
    default:
      return kernel == CM_CUBE ? run(radius_tile_kernel<CM_MIXED, MODE, 1>)
                               : run(radius_tile_kernel<CM_MIXED, MODE, 0>);
  }
}

}  // namespace

void query_stats(uint64_t* out, int reset) {
  unsigned long long h[4];
  cudaMemcpyFromSymbol(h, g_qstats, sizeof(h));
  for (int i = 0; i < 4; ++i) out[i] = h[i];
  if (reset) {
    const unsigned long long z[4] = {0, 0, 0, 0};
    cudaMemcpyToSymbol(g_qstats, z, sizeof(z));
  }
}

cm_status order_queries(const cm_index* ix, const double* q, uint64_t nq, cudaStream_t st,
                        QueryOrder* out) {
  out->nq = nq;
  out->st = st;
  if (nq == 0) return CM_OK;
  CM_CUDA_TRY(dev_alloc_t(&out->perm, nq, st));
  return ix->V <= (1ull << 32) ? order_typed<uint32_t>(ix, q, nq, st, out->perm)
                               : order_typed<uint64_t>(ix, q, nq, st, out->perm);
}

cm_status radius_count_dev(const cm_index* ix, const double* q, uint64_t nq, int kernel, double r,
                           const uint32_t* perm, uint32_t* counts, uint64_t* tested,
                           cudaStream_t st) {
  if (nq == 0) return CM_OK;
  return launch_radius<MODE_COUNT>(ix, q, nq, kernel, r, perm, counts, tested, nullptr, nullptr,
                                   nullptr, nullptr, nullptr, st);
}

cm_status radius_digest_dev(const cm_index* ix, const double* q, uint64_t nq, int kernel, double r,
                            const uint32_t* perm, uint32_t* counts, uint64_t* digests,
                            cudaStream_t st) {
  if (nq == 0) return CM_OK;
  return launch_radius<MODE_DIGEST>(ix, q, nq, kernel, r, perm, counts, nullptr, digests, nullptr,
                                    nullptr, nullptr, nullptr, st);
}

cm_status radius_fill_dev(const cm_index* ix, const double* q, uint64_t nq, int kernel, double r,
                          const uint32_t* perm, const uint64_t* row_ptr, uint32_t* cols,
                          cudaStream_t st, cudaEvent_t after_fill) {
  if (nq == 0) return CM_OK;
  uint32_t* big = nullptr;
  uint32_t* nbig = nullptr;
  CM_CUDA_TRY(dev_alloc_t(&big, nq, st));
  CM_CUDA_TRY(dev_alloc_t(&nbig, 1, st));
  CM_CUDA_TRY(cudaMemsetAsync(nbig, 0, 4, st));
  cm_status s = launch_radius<MODE_FILL>(ix, q, nq, kernel, r, perm, nullptr, nullptr, nullptr,
                                         row_ptr, cols, big, nbig, st);
  if (after_fill) cudaEventRecord(after_fill, st);
  if (s == CM_OK) {
    static bool configured = false;
    const int smem = kBigSmemCap * 4;
    if (!configured) {
      cudaFuncSetAttribute(big_row_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      configured = true;
    }
    big_row_sort_kernel<<<sm_count(), 1024, smem, st>>>(row_ptr, cols, big, nbig); ::cmg::note_launch();
    if (cudaGetLastError() != cudaSuccess) {
      set_error("big_row_sort_kernel launch failed");
      s = CM_CUDA;
    }
  }
  dev_free(big, st);
  dev_free(nbig, st);
  return s;
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
