// Warp-uniform record streaming shared by the query-tile kernels (radius
// tiles in query.cu, kNN tiles in knn.cu): column spans staged into shared
// memory by cp.async one chunk ahead, read by every lane of the warp.
#pragma once

#include "common.cuh"
#include "filter.cuh"

namespace cmg {
namespace tw {

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

// A staged record as read from shared memory: xyz, handle, voxel k.
struct __align__(16) SRec {
  double x, y, z;
  uint32_t id, meta;
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Records [p, p + len) -> stg[0..len): lane t copies record t (2 x 16 B).
__device__ __forceinline__ void stage_chunk(PointRec* stg, const PointRec* rec, uint32_t p,
                                            uint32_t len, int lane) {
  if ((uint32_t)lane < len) {
    const char* g = reinterpret_cast<const char*>(rec + p + lane);
    char* d = reinterpret_cast<char*>(stg + lane);
    cp_async16(d, g);
    cp_async16(d + 16, g + 16);
  }
}

// Float records [p, p + len) -> stg[0..len): lane t copies record t (16 B).
__device__ __forceinline__ void stage_chunk_f(FRec* stg, const FRec* frec, uint32_t p,
                                              uint32_t len, int lane) {
  if ((uint32_t)lane < len) cp_async16(stg + lane, frec + p + lane);
}

// Chunk iterator over the hull's needed columns (bit c of `mask`), spans
// [b_c, e_c) held by lane c. `first` starts at the lowest needed column;
// otherwise moves past the chunk [p, p + 32) of column c. Warp-uniform.
__device__ __forceinline__ bool advance_chunk(uint32_t& mask, uint32_t& c, uint32_t& p,
                                              uint32_t& ce, uint32_t b, uint32_t e, bool first) {
  if (!first) {
    if (p + 32 < ce) {
      p += 32;
      return true;
    }
    mask &= ~(1u << c);
  }
  while (mask) {
    c = __ffs(mask) - 1;
    p = __shfl_sync(0xffffffffu, b, c);
    ce = __shfl_sync(0xffffffffu, e, c);
    if (p < ce) return true;
    mask &= ~(1u << c);
  }
  return false;
}

}  // namespace tw
}  // namespace cmg
