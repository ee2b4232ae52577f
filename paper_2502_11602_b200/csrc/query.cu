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

constexpr int kQThreads = 256;
constexpr int kQWarps = kQThreads / 32;
constexpr int kRowCap = 2048;      // per-warp row buffer (u32 entries)
constexpr int kBigSmemCap = 32768;  // block sort in shared memory (128 KB)

enum { MODE_COUNT = 0, MODE_FILL = 1, MODE_DIGEST = 2 };

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

template <int FLAVOR, int MODE>
__global__ void __launch_bounds__(kQThreads) radius_warp_kernel(
    const Tables t, const double* __restrict__ q, uint64_t nq, double r, int cube,
    const uint32_t* __restrict__ perm, uint32_t* __restrict__ counts,
    uint64_t* __restrict__ tested, uint64_t* __restrict__ digests,
    const uint64_t* __restrict__ row_ptr, uint32_t* __restrict__ cols,
    uint32_t* __restrict__ big_rows, uint32_t* __restrict__ n_big) {
  extern __shared__ uint32_t sbuf[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const uint64_t W = (uint64_t)gridDim.x * kQWarps;
  const uint32_t lt = lanemask_lt();
  uint32_t* wbuf = sbuf + wib * kRowCap;

  for (uint64_t s = (uint64_t)blockIdx.x * kQWarps + wib; s < nq; s += W) {
    const uint32_t qi = perm ? __ldg(perm + s) : (uint32_t)s;
    const double cx = __ldg(q + 3 * (uint64_t)qi);
    const double cy = __ldg(q + 3 * (uint64_t)qi + 1);
    const double cz = __ldg(q + 3 * (uint64_t)qi + 2);
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
      __syncwarp();
    }
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
  const size_t smem = MODE == MODE_FILL ? (size_t)kQWarps * kRowCap * 4 : 0;
  auto run = [&](auto kern) -> cm_status {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kQThreads, smem);
    per_sm = std::max(per_sm, 1);
    const uint64_t need = (nq + kQWarps - 1) / kQWarps;
    const unsigned grid =
        (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(need, (uint64_t)sm_count() * per_sm));
    kern<<<grid, kQThreads, smem, st>>>(t, q, nq, r, kernel == CM_CUBE, perm, counts, tested,
                                        digests, row_ptr, cols, big_rows, n_big); ::cmg::note_launch();
    CM_CUDA_TRY(cudaGetLastError());
    return CM_OK;
  };
  switch (ix->opts.flavor) {
    case CM_DENSE: return run(radius_warp_kernel<CM_DENSE, MODE>);
    case CM_SPARSE: return run(radius_warp_kernel<CM_SPARSE, MODE>);
    default: return run(radius_warp_kernel<CM_MIXED, MODE>);
  }
}

}  // namespace

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
