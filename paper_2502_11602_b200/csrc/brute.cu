// Brute-force baselines on sm_100a — brute_radius (baseline.hpp:11-21) and
// brute_knn (baseline.cpp:8-25): every point against every centre, no index.
// They back the CLI's `verify` (tools/cmd_verify.cpp:31-114) on the device:
// the index-based kernels must agree with a linear scan.
//
// brute_radius: one block per centre, 256 threads stride over the points and
// test the kernel predicate with the reference's arithmetic (the same
// `Predicate` as the index path); the set is reported as (count,
// Σ splitmix64(handle)), the digest cm_radius_digest produces.
// brute_knn: one block per centre; each thread keeps the k smallest
// (d², handle) of its stride in a local sorted list, then the block extracts
// the k smallest of the 256 lists, one block-wide argmin per output.
#include "index.cuh"
#include "sort_scan.cuh"

namespace cmg {

int sm_count();

namespace {

constexpr int kBruteThreads = 256;

__device__ __forceinline__ bool brute_pred(int kind, const Predicate& P, double x, double y,
                                           double z) {
  if (kind == 1)
    return (x >= P.lx) & (x <= P.hx) & (y >= P.ly) & (y <= P.hy) & (z >= P.lz) & (z <= P.hz);
  if (kind == 2) {
    const double dx = __dsub_rn(x, P.cx), dy = __dsub_rn(y, P.cy);
    return (z >= P.lz) & (z <= P.hz) & (__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)) <= P.rr);
  }
  return sqdist(x, y, z, P.cx, P.cy, P.cz) <= P.rr;
}

__global__ void __launch_bounds__(kBruteThreads) brute_radius_kernel(
    const double* __restrict__ xyz, uint64_t n, const double* __restrict__ q, uint64_t nq,
    int kind, double r, uint32_t* __restrict__ counts, uint64_t* __restrict__ digests) {
  __shared__ uint32_t sc[kBruteThreads / 32];
  __shared__ unsigned long long sd[kBruteThreads / 32];
  for (uint64_t qi = blockIdx.x; qi < nq; qi += gridDim.x) {
    Predicate P;
    P.init(q[3 * qi], q[3 * qi + 1], q[3 * qi + 2], r, kind);
    uint32_t cnt = 0;
    uint64_t dig = 0;
    for (uint64_t h = threadIdx.x; h < n; h += kBruteThreads) {
      if (brute_pred(kind, P, __ldg(xyz + 3 * h), __ldg(xyz + 3 * h + 1), __ldg(xyz + 3 * h + 2))) {
        ++cnt;
        dig += mix64(h);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
      dig += __shfl_xor_sync(0xffffffffu, dig, o);
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) sc[w] = cnt, sd[w] = dig;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t c = 0;
      uint64_t d = 0;
      for (int i = 0; i < kBruteThreads / 32; ++i) c += sc[i], d += sd[i];
      counts[qi] = c;
      digests[qi] = d;
    }
    __syncthreads();
  }
}

__device__ __forceinline__ bool pair_lt(double a, uint32_t ia, double b, uint32_t ib) {
  return a < b || (a == b && ia < ib);
}

__global__ void __launch_bounds__(kBruteThreads) brute_knn_kernel(
    const double* __restrict__ xyz, uint64_t n, const double* __restrict__ q, uint64_t nq,
    uint32_t k, uint32_t* __restrict__ idx_out, double* __restrict__ d2_out) {
  __shared__ double rd[kBruteThreads / 32];
  __shared__ uint32_t ri[kBruteThreads / 32];
  __shared__ int rt[kBruteThreads / 32];
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);
  for (uint64_t qi = blockIdx.x; qi < nq; qi += gridDim.x) {
    const double cx = q[3 * qi], cy = q[3 * qi + 1], cz = q[3 * qi + 2];
    double ld[kBruteKMax];
    uint32_t li[kBruteKMax];
    uint32_t cnt = 0;
    for (uint64_t h = threadIdx.x; h < n; h += kBruteThreads) {
      const double d2 = sqdist(__ldg(xyz + 3 * h), __ldg(xyz + 3 * h + 1), __ldg(xyz + 3 * h + 2),
                               cx, cy, cz);
      const uint32_t id = (uint32_t)h;
      if (cnt == k && !pair_lt(d2, id, ld[k - 1], li[k - 1])) continue;
      uint32_t pos = cnt < k ? cnt : k - 1;  // insertion from the back
      while (pos > 0 && pair_lt(d2, id, ld[pos - 1], li[pos - 1])) {
        ld[pos] = ld[pos - 1];
        li[pos] = li[pos - 1];
        --pos;
      }
      ld[pos] = d2;
      li[pos] = id;
      if (cnt < k) ++cnt;
    }
    // k rounds of block-wide argmin over the lists' heads
    uint32_t head = 0;
    for (uint32_t out = 0; out < k; ++out) {
      double bd = head < cnt ? ld[head] : kInf;
      uint32_t bi = head < cnt ? li[head] : 0xffffffffu;
      int bt = head < cnt ? (int)threadIdx.x : -1;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double od = __shfl_xor_sync(0xffffffffu, bd, o);
        const uint32_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
        const int ot = __shfl_xor_sync(0xffffffffu, bt, o);
        if (ot >= 0 && (bt < 0 || pair_lt(od, oi, bd, bi))) bd = od, bi = oi, bt = ot;
      }
      const int w = threadIdx.x >> 5;
      if ((threadIdx.x & 31) == 0) rd[w] = bd, ri[w] = bi, rt[w] = bt;
      __syncthreads();
      if (threadIdx.x == 0) {
        for (int i = 1; i < kBruteThreads / 32; ++i)
          if (rt[i] >= 0 && (rt[0] < 0 || pair_lt(rd[i], ri[i], rd[0], ri[0])))
            rd[0] = rd[i], ri[0] = ri[i], rt[0] = rt[i];
        idx_out[qi * k + out] = rt[0] >= 0 ? ri[0] : 0xffffffffu;
        d2_out[qi * k + out] = rt[0] >= 0 ? rd[0] : kInf;
      }
      __syncthreads();
      if ((int)threadIdx.x == rt[0]) ++head;
      __syncthreads();
    }
  }
}

// One warp per CSR row: count, Σ splitmix64(handle) (the cm_radius_digest
// digest) and whether the row is strictly ascending.
__global__ void __launch_bounds__(256) csr_digest_kernel(const uint64_t* __restrict__ row_ptr,
                                                         const uint32_t* __restrict__ cols,
                                                         uint64_t nq, uint32_t* __restrict__ counts,
                                                         uint64_t* __restrict__ digests,
                                                         unsigned long long* __restrict__ unsorted) {
  const int lane = threadIdx.x & 31;
  const uint64_t W = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t q = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); q < nq; q += W) {
    const uint64_t b = row_ptr[q], e = row_ptr[q + 1];
    uint64_t dig = 0;
    bool bad = e < b;
    for (uint64_t i = b + lane; i < e; i += 32) {
      const uint32_t v = cols[i];
      dig += mix64(v);
      if (i > b && cols[i - 1] >= v) bad = true;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dig += __shfl_xor_sync(0xffffffffu, dig, o);
    bad = __any_sync(0xffffffffu, bad);
    if (lane == 0) {
      if (counts) counts[q] = (uint32_t)(e - b);
      if (digests) digests[q] = dig;
      if (bad) atomicAdd(unsorted, 1ull);
    }
  }
}

}  // namespace

cm_status csr_digest_dev(const uint64_t* row_ptr, const uint32_t* cols, uint64_t nq,
                         uint32_t* counts, uint64_t* digests, unsigned long long* unsorted,
                         cudaStream_t st) {
  CM_CUDA_TRY(cudaMemsetAsync(unsorted, 0, 8, st));
  if (nq == 0) return CM_OK;
  const unsigned grid = (unsigned)std::min<uint64_t>((nq + 7) / 8, (uint64_t)sm_count() * 16);
  csr_digest_kernel<<<grid, 256, 0, st>>>(row_ptr, cols, nq, counts, digests, unsorted); note_launch();
  CM_CUDA_TRY(cudaGetLastError());
  return CM_OK;
}

cm_status brute_radius_dev(const double* xyz, uint64_t n, const double* q, uint64_t nq, int kind,
                           double r, uint32_t* counts, uint64_t* digests, cudaStream_t st) {
  if (nq == 0) return CM_OK;
  const unsigned grid = (unsigned)std::min<uint64_t>(nq, (uint64_t)sm_count() * 8);
  brute_radius_kernel<<<grid, kBruteThreads, 0, st>>>(xyz, n, q, nq, kind, r, counts, digests); note_launch();
  CM_CUDA_TRY(cudaGetLastError());
  return CM_OK;
}

cm_status brute_knn_dev(const double* xyz, uint64_t n, const double* q, uint64_t nq, uint32_t k,
                        uint32_t* idx, double* d2, cudaStream_t st) {
  if (nq == 0) return CM_OK;
  const unsigned grid = (unsigned)std::min<uint64_t>(nq, (uint64_t)sm_count() * 8);
  brute_knn_kernel<<<grid, kBruteThreads, 0, st>>>(xyz, n, q, nq, k, idx, d2); note_launch();
  CM_CUDA_TRY(cudaGetLastError());
  return CM_OK;
}

}  // namespace cmg
