// In-house device primitives: exclusive scan and a stable LSD radix sort of
// (key, u32 value) pairs. The sort replaces the reference's
// std::stable_sort by cell key (map.cpp:51-54) and its counting sort
// (map.cpp:67-81): LSD radix sort is stable, and the values start as iota,
// so the permutation equals the reference's stable_sort permutation.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "common.cuh"

namespace cmg {

int sm_count();

// ------------------------------------------------------------------ scan --

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T u = __shfl_up_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) >= o) v += u;
  }
  return v;
}

// Block-wide exclusive scan of one value per thread; returns the block total.
template <typename T>
__device__ __forceinline__ T block_excl_scan(T v, T* smem_warp /*[32]*/, T* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const T inc = warp_incl_scan(v);
  if (lane == 31) smem_warp[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    T w = lane < nw ? smem_warp[lane] : T(0);
    const T wi = warp_incl_scan(w);
    smem_warp[lane] = wi - w;
    if (lane == 31) smem_warp[32] = wi;
  }
  __syncthreads();
  const T out = smem_warp[wid] + inc - v;
  *total = smem_warp[32];
  __syncthreads();
  return out;
}

template <typename TI, typename TO>
__global__ void scan_reduce_kernel(const TI* __restrict__ in, uint64_t n, TO* __restrict__ part) {
  __shared__ TO sw[33];
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile;
  TO s = 0;
#pragma unroll
  for (int it = 0; it < kScanItems; ++it) {
    const uint64_t i = base + (uint64_t)it * kScanThreads + threadIdx.x;
    if (i < n) s += (TO)in[i];
  }
  TO tot;
  block_excl_scan<TO>(s, sw, &tot);
  if (threadIdx.x == 0) part[blockIdx.x] = tot;
}

// Single block: exclusive scan of the per-tile partial sums, in place.
template <typename TO>
__global__ void scan_partials_kernel(TO* part, uint64_t nb) {
  __shared__ TO sw[33];
  TO carry = 0;
  for (uint64_t base = 0; base < nb; base += blockDim.x) {
    const uint64_t i = base + threadIdx.x;
    const TO v = i < nb ? part[i] : TO(0);
    TO tot;
    const TO ex = block_excl_scan<TO>(v, sw, &tot);
    if (i < nb) part[i] = carry + ex;
    carry += tot;
  }
}

// out[i] = sum(in[0..i)) ; if total != nullptr, out[n] = total as well when
// write_total is set.
template <typename TI, typename TO>
__global__ void scan_apply_kernel(const TI* __restrict__ in, uint64_t n, const TO* __restrict__ part,
                                  TO* __restrict__ out, int write_total) {
  __shared__ TO sw[33];
  __shared__ TO tile_vals[kScanTile];
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile;
  // blocked arrangement in smem: thread t owns items t*ITEMS .. +ITEMS
  for (int it = 0; it < kScanItems; ++it) {
    const uint64_t i = base + (uint64_t)it * kScanThreads + threadIdx.x;
    tile_vals[it * kScanThreads + threadIdx.x] = i < n ? (TO)in[i] : TO(0);
  }
  __syncthreads();
  TO loc[kScanItems];
  TO s = 0;
#pragma unroll
  for (int it = 0; it < kScanItems; ++it) {
    loc[it] = tile_vals[threadIdx.x * kScanItems + it];
    s += loc[it];
  }
  TO tot;
  TO ex = block_excl_scan<TO>(s, sw, &tot) + part[blockIdx.x];
#pragma unroll
  for (int it = 0; it < kScanItems; ++it) {
    tile_vals[threadIdx.x * kScanItems + it] = ex;
    ex += loc[it];
  }
  __syncthreads();
  for (int it = 0; it < kScanItems; ++it) {
    const uint64_t i = base + (uint64_t)it * kScanThreads + threadIdx.x;
    if (i < n) out[i] = tile_vals[it * kScanThreads + threadIdx.x];
  }
  if (write_total && blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {
    out[n] = part[blockIdx.x] + tot;
  }
}

// Exclusive scan of n inputs into out[0..n) (+ out[n] = total when
// write_total). `part` scratch needs ceil(n / kScanTile) entries.
template <typename TI, typename TO>
inline void exclusive_scan(const TI* in, uint64_t n, TO* out, TO* part, int write_total,
                           cudaStream_t st) {
  const uint64_t nb = (n + kScanTile - 1) / kScanTile;
  if (nb == 0) {
    if (write_total) cudaMemsetAsync(out, 0, sizeof(TO), st);
    return;
  }
  scan_reduce_kernel<TI, TO><<<(unsigned)nb, kScanThreads, 0, st>>>(in, n, part); ::cmg::note_launch();
  scan_partials_kernel<TO><<<1, 1024, 0, st>>>(part, nb); ::cmg::note_launch();
  scan_apply_kernel<TI, TO><<<(unsigned)nb, kScanThreads, 0, st>>>(in, n, part, out, write_total); ::cmg::note_launch();
}

inline uint64_t scan_part_elems(uint64_t n) { return (n + kScanTile - 1) / kScanTile + 1; }

// ------------------------------------------------------------ radix sort --

constexpr int kSortThreads = 256;  // 8 warps
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kSortItems = 16;  // per lane; a warp owns 512 consecutive keys
constexpr int kSortTile = kSortThreads * kSortItems;
constexpr int kRadixBitsMax = 10;  // digits of 8..10 bits (wcount fits static smem)
constexpr int kRadixMax = 1 << kRadixBitsMax;

// Per-block digit counts. Each warp counts into its own shared histogram
// (the low-digit passes see few distinct digits per block, and one shared
// histogram serialised its atomics), all loads issued before the first count.
template <typename K, int RB>
__global__ void __launch_bounds__(kSortThreads) radix_upsweep(const K* __restrict__ keys,
                                                              uint64_t n, int shift,
                                                              uint32_t* __restrict__ hist,
                                                              uint32_t nblocks) {
  constexpr int kRadix = 1 << RB;
  __shared__ uint32_t h[kSortWarps][kRadix];
  const int w = threadIdx.x >> 5;
  for (int d = threadIdx.x; d < kSortWarps * kRadix; d += blockDim.x) (&h[0][0])[d] = 0;
  __syncthreads();
  const uint64_t base = (uint64_t)blockIdx.x * kSortTile;
  K kv[kSortItems];
#pragma unroll
  for (int it = 0; it < kSortItems; ++it) {
    const uint64_t i = base + (uint64_t)it * kSortThreads + threadIdx.x;
    kv[it] = i < n ? keys[i] : K(0);
  }
#pragma unroll
  for (int it = 0; it < kSortItems; ++it) {
    const uint64_t i = base + (uint64_t)it * kSortThreads + threadIdx.x;
    if (i < n) atomicAdd(&h[w][(uint32_t)(kv[it] >> shift) & (kRadix - 1)], 1u);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < kRadix; d += blockDim.x) {
    uint32_t s = 0;
#pragma unroll
    for (int ww = 0; ww < kSortWarps; ++ww) s += h[ww][d];
    hist[(uint64_t)d * nblocks + blockIdx.x] = s;
  }
}

// Stable scatter. Warp w of block b owns keys [b*TILE + w*512, +512);
// item `it` of lane l is key (it*32 + l) of that run, so processing items in
// order with lanes in order visits keys in input order. Ranks inside a warp
// come from __match_any_sync peer groups. The block first reorders its tile
// by digit in shared memory (stable: warp, then rank), then writes it out in
// that order, so consecutive threads store consecutive positions of one
// digit's run (a few sectors per digit) instead of one sector per key.
template <typename K, int RB>
struct DownsweepSmem {
  static constexpr int kRadix = 1 << RB;
  uint32_t wcount[kSortWarps][kRadix];
  uint32_t lbase[kRadix];
  uint32_t goff[kRadix];
  uint32_t swarp[33];
  K skeys[kSortTile];
  uint32_t svals[kSortTile];
};

template <typename K, int RB>
__global__ void __launch_bounds__(kSortThreads) radix_downsweep(
    const K* __restrict__ keys_in, const uint32_t* __restrict__ vals_in, K* __restrict__ keys_out,
    uint32_t* __restrict__ vals_out, uint64_t n, int shift,
    const uint32_t* __restrict__ offs /* scanned hist [d][b] */, uint32_t nblocks) {
  constexpr int kRadix = 1 << RB;
  constexpr int kPer = kRadix / kSortThreads > 0 ? kRadix / kSortThreads : 1;
  static_assert(kRadix % kSortThreads == 0, "digits per thread");
  extern __shared__ __align__(16) unsigned char dsm_raw[];
  DownsweepSmem<K, RB>& sm = *reinterpret_cast<DownsweepSmem<K, RB>*>(dsm_raw);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int d = lane; d < kRadix; d += 32) sm.wcount[w][d] = 0;
  __syncwarp();
  const uint64_t bbase = (uint64_t)blockIdx.x * kSortTile;
  const uint64_t wbase = bbase + (uint64_t)w * (32 * kSortItems);
  K kv[kSortItems];
  uint32_t vv[kSortItems];
  uint32_t rank[kSortItems];
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int it = 0; it < kSortItems; ++it) {  // all loads in flight first
    const uint64_t i = wbase + (uint64_t)it * 32 + lane;
    const bool valid = i < n;
    kv[it] = valid ? keys_in[i] : K(0);
    vv[it] = valid ? vals_in[i] : 0u;
  }
  // Stable ranks: items in order; the lowest lane of each digit's peer group
  // bumps the warp's digit counter with one shared-memory atomic (the warp's
  // atomics are performed in issue order) and hands the old count to its peers.
#pragma unroll
  for (int it = 0; it < kSortItems; ++it) {
    const uint64_t i = wbase + (uint64_t)it * 32 + lane;
    const bool valid = i < n;
    const uint32_t d = valid ? ((uint32_t)(kv[it] >> shift) & (kRadix - 1)) : kRadix;  // kRadix = invalid
#ifndef CM_RADIX_MATCH_ANY
    // peer group by one ballot per digit bit (invalid lanes drop out first);
    // measured faster than __match_any_sync (20M-key sort 0.83 -> 0.75 ms)
    uint32_t peers = __ballot_sync(0xffffffffu, valid);
#pragma unroll
    for (int b = 0; b < RB; ++b) {
      const bool bit = (d >> b) & 1u;
      const uint32_t m = __ballot_sync(0xffffffffu, bit);
      peers &= bit ? m : ~m;
    }
    if (!valid) peers = 1u << lane;
#else
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
#endif
    const int leader = __ffs(peers) - 1;
    uint32_t old = 0;
    if (valid && lane == leader) old = atomicAdd(&sm.wcount[w][d], (uint32_t)__popc(peers));
    old = __shfl_sync(0xffffffffu, old, leader);
    rank[it] = old + __popc(peers & lt);
  }
  __syncwarp();
  __syncthreads();
  // per digit: exclusive prefix over warps (in place), the block's total,
  // its global offset; then the block-local digit starts (scan over digits)
  uint32_t tsum = 0;
#pragma unroll
  for (int x = 0; x < kPer; ++x) {
    const int d = threadIdx.x * kPer + x;
    uint32_t s2 = 0;
    for (int ww = 0; ww < kSortWarps; ++ww) {
      const uint32_t c = sm.wcount[ww][d];
      sm.wcount[ww][d] = s2;
      s2 += c;
    }
    sm.lbase[d] = s2;  // total for now
    sm.goff[d] = offs[(uint64_t)d * nblocks + blockIdx.x];
    tsum += s2;
  }
  uint32_t btot;
  uint32_t run = block_excl_scan<uint32_t>(tsum, sm.swarp, &btot);
#pragma unroll
  for (int x = 0; x < kPer; ++x) {
    const int d = threadIdx.x * kPer + x;
    const uint32_t c = sm.lbase[d];
    sm.lbase[d] = run;
    run += c;
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < kSortItems; ++it) {
    const uint64_t i = wbase + (uint64_t)it * 32 + lane;
    if (i < n) {
      const uint32_t d = (uint32_t)(kv[it] >> shift) & (kRadix - 1);
      const uint32_t lpos = sm.lbase[d] + sm.wcount[w][d] + rank[it];
      sm.skeys[lpos] = kv[it];
      sm.svals[lpos] = vv[it];
    }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < btot; i += kSortThreads) {
    const K key = sm.skeys[i];
    const uint32_t d = (uint32_t)(key >> shift) & (kRadix - 1);
    const uint32_t pos = sm.goff[d] + (i - sm.lbase[d]);
    keys_out[pos] = key;
    vals_out[pos] = sm.svals[i];
  }
}

// ---- onesweep-style passes: one global histogram kernel for every digit
// position, then one kernel per pass whose tiles find their digits' global
// offsets by decoupled look-back (no per-pass upsweep and scan) -----------
//
// Digit histograms of every pass at once: per-warp private shared-memory
// counters (low-digit passes hit few distinct digits per block, which
// serialised the single shared histogram's atomics), summed into
// ghist[pass][digit] with one global atomic per (block, pass, digit).
template <typename K, int RB>
__global__ void __launch_bounds__(kSortThreads) radix_hist_all(const K* __restrict__ keys,
                                                               uint64_t n, int passes,
                                                               uint32_t* __restrict__ ghist) {
  constexpr int kRadix = 1 << RB;
  extern __shared__ uint32_t hh[];  // [passes][kSortWarps][kRadix]
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < passes * kSortWarps * kRadix; i += blockDim.x) hh[i] = 0;
  __syncthreads();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const K key = keys[i];
    for (int p = 0; p < passes; ++p)
      atomicAdd(&hh[(p * kSortWarps + w) * kRadix + ((uint32_t)(key >> (p * RB)) & (kRadix - 1))], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * kRadix; i += blockDim.x) {
    const int p = i / kRadix, d = i % kRadix;
    uint32_t s = 0;
    for (int ww = 0; ww < kSortWarps; ++ww) s += hh[(p * kSortWarps + ww) * kRadix + d];
    if (s) atomicAdd(&ghist[i], s);
  }
  (void)lane;
}

// ghist[pass][d] -> exclusive prefix over d, in place (one block per pass).
template <int RB>
__global__ void radix_digit_starts(uint32_t* __restrict__ ghist) {
  constexpr int kRadix = 1 << RB;
  constexpr int kPer = kRadix / kSortThreads;
  __shared__ uint32_t sw[33];
  uint32_t* h = ghist + (size_t)blockIdx.x * kRadix;
  uint32_t v[kPer], s = 0;
#pragma unroll
  for (int x = 0; x < kPer; ++x) {
    v[x] = h[threadIdx.x * kPer + x];
    s += v[x];
  }
  uint32_t tot;
  uint32_t run = block_excl_scan<uint32_t>(s, sw, &tot);
#pragma unroll
  for (int x = 0; x < kPer; ++x) {
    h[threadIdx.x * kPer + x] = run;
    run += v[x];
  }
}

// Look-back status word per (tile, digit): bits 31..30 = 0 empty, 1 the
// tile's own count, 2 the inclusive prefix through the tile; bits 29..0 the
// value (n < 2^30). Value and flag share one word, so a plain volatile
// store publishes both.
constexpr uint32_t kLbAgg = 1u << 30, kLbInc = 2u << 30, kLbMask = (1u << 30) - 1;

template <typename K, int RB>
__global__ void __launch_bounds__(kSortThreads) radix_onesweep(
    const K* __restrict__ keys_in, const uint32_t* __restrict__ vals_in, K* __restrict__ keys_out,
    uint32_t* __restrict__ vals_out, uint64_t n, int shift,
    const uint32_t* __restrict__ dstart /* [kRadix] */, uint32_t* status /* [tiles][kRadix] */,
    uint32_t* tile_ctr) {
  constexpr int kRadix = 1 << RB;
  constexpr int kPer = kRadix / kSortThreads > 0 ? kRadix / kSortThreads : 1;
  static_assert(kRadix % kSortThreads == 0, "digits per thread");
  extern __shared__ __align__(16) unsigned char dsm_raw[];
  DownsweepSmem<K, RB>& sm = *reinterpret_cast<DownsweepSmem<K, RB>*>(dsm_raw);
  __shared__ uint32_t s_tile;
  // tiles are numbered in launch order, so every predecessor a tile looks
  // back at has started (and will publish): no deadlock
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int d = lane; d < kRadix; d += 32) sm.wcount[w][d] = 0;
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t bbase = (uint64_t)tile * kSortTile;
  const uint64_t wbase = bbase + (uint64_t)w * (32 * kSortItems);
  K kv[kSortItems];
  uint32_t vv[kSortItems];
  uint32_t rank[kSortItems];
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int it = 0; it < kSortItems; ++it) {
    const uint64_t i = wbase + (uint64_t)it * 32 + lane;
    const bool valid = i < n;
    kv[it] = valid ? keys_in[i] : K(0);
    vv[it] = valid ? vals_in[i] : 0u;
  }
#pragma unroll
  for (int it = 0; it < kSortItems; ++it) {
    const uint64_t i = wbase + (uint64_t)it * 32 + lane;
    const bool valid = i < n;
    const uint32_t d = valid ? ((uint32_t)(kv[it] >> shift) & (kRadix - 1)) : kRadix;
    uint32_t peers = __ballot_sync(0xffffffffu, valid);
#pragma unroll
    for (int b = 0; b < RB; ++b) {
      const bool bit = (d >> b) & 1u;
      const uint32_t m = __ballot_sync(0xffffffffu, bit);
      peers &= bit ? m : ~m;
    }
    if (!valid) peers = 1u << lane;
    const int leader = __ffs(peers) - 1;
    uint32_t old = 0;
    if (valid && lane == leader) old = atomicAdd(&sm.wcount[w][d], (uint32_t)__popc(peers));
    old = __shfl_sync(0xffffffffu, old, leader);
    rank[it] = old + __popc(peers & lt);
  }
  __syncwarp();
  __syncthreads();
  uint32_t tsum = 0;
  uint32_t cnt[kPer];
#pragma unroll
  for (int x = 0; x < kPer; ++x) {
    const int d = threadIdx.x * kPer + x;
    uint32_t s2 = 0;
    for (int ww = 0; ww < kSortWarps; ++ww) {
      const uint32_t c = sm.wcount[ww][d];
      sm.wcount[ww][d] = s2;
      s2 += c;
    }
    cnt[x] = s2;
    sm.lbase[d] = s2;
    tsum += s2;
    // publish this tile's count at once, the prefix after the look-back
    volatile uint32_t* st = status + (size_t)tile * kRadix + d;
    *st = (tile == 0 ? kLbInc : kLbAgg) | s2;
  }
#pragma unroll
  for (int x = 0; x < kPer; ++x) {
    const int d = threadIdx.x * kPer + x;
    uint32_t excl = 0;
    if (tile > 0) {
      for (int64_t tt = (int64_t)tile - 1; tt >= 0; --tt) {
        const volatile uint32_t* sp = status + (size_t)tt * kRadix + d;
        uint32_t v;
        do {
          v = *sp;
        } while ((v & ~kLbMask) == 0);
        excl += v & kLbMask;
        if (v & kLbInc) break;
      }
      volatile uint32_t* st = status + (size_t)tile * kRadix + d;
      *st = kLbInc | (excl + cnt[x]);
    }
    sm.goff[d] = dstart[d] + excl;
  }
  uint32_t btot;
  uint32_t run = block_excl_scan<uint32_t>(tsum, sm.swarp, &btot);
#pragma unroll
  for (int x = 0; x < kPer; ++x) {
    const int d = threadIdx.x * kPer + x;
    const uint32_t c = sm.lbase[d];
    sm.lbase[d] = run;
    run += c;
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < kSortItems; ++it) {
    const uint64_t i = wbase + (uint64_t)it * 32 + lane;
    if (i < n) {
      const uint32_t d = (uint32_t)(kv[it] >> shift) & (kRadix - 1);
      const uint32_t lpos = sm.lbase[d] + sm.wcount[w][d] + rank[it];
      sm.skeys[lpos] = kv[it];
      sm.svals[lpos] = vv[it];
    }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < btot; i += kSortThreads) {
    const K key = sm.skeys[i];
    const uint32_t d = (uint32_t)(key >> shift) & (kRadix - 1);
    const uint32_t pos = sm.goff[d] + (i - sm.lbase[d]);
    keys_out[pos] = key;
    vals_out[pos] = sm.svals[i];
  }
}

template <typename K, int RB>
inline void launch_onesweep(const K* ka, const uint32_t* va, K* kb, uint32_t* vb, uint64_t n,
                            int shift, const uint32_t* dstart, uint32_t* status,
                            uint32_t* tile_ctr, uint32_t nb, cudaStream_t st) {
  const int smem = (int)sizeof(DownsweepSmem<K, RB>);
  cudaFuncSetAttribute(radix_onesweep<K, RB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  radix_onesweep<K, RB><<<nb, kSortThreads, smem, st>>>(ka, va, kb, vb, n, shift, dstart, status,
                                                         tile_ctr);
  ::cmg::note_launch();
}

template <typename K, int RB>
inline void launch_downsweep(const K* ka, const uint32_t* va, K* kb, uint32_t* vb, uint64_t n,
                             int shift, const uint32_t* hist, uint32_t nb, cudaStream_t st) {
  const int smem = (int)sizeof(DownsweepSmem<K, RB>);
  cudaFuncSetAttribute(radix_downsweep<K, RB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  radix_downsweep<K, RB><<<nb, kSortThreads, smem, st>>>(ka, va, kb, vb, n, shift, hist, nb);
  ::cmg::note_launch();
}

// Scratch (bytes) for radix_sort_pairs over n keys.
template <typename K>
inline size_t radix_scratch_bytes(uint64_t n) {
  const uint64_t nb = (n + kSortTile - 1) / kSortTile;
  const uint64_t h = nb * kRadixMax;
  // + the onesweep passes' digit histograms and tile counters (8 passes max)
  return (size_t)(n * (sizeof(K) + 4)) + (size_t)(h * 4) + (size_t)(scan_part_elems(h) * 4) +
         (size_t)(8 * kRadixMax + 8) * 4 + 256;
}

// Sorts (keys, vals) by the low `bits` bits of the keys, stably. n < 2^32.
// Result ends in (keys, vals) (the function ping-pongs through scratch).
// Returns the number of passes.
// kres / vres (optional): receive where the sorted pairs are (keys / vals or
// the scratch copy) instead of copying an odd pass count's result back.
template <typename K>
inline int radix_sort_pairs(K* keys, uint32_t* vals, uint64_t n, int bits, void* scratch,
                            cudaStream_t st, K** kres = nullptr, uint32_t** vres = nullptr) {
  if (kres) *kres = keys;
  if (vres) *vres = vals;
  if (n <= 1 || bits <= 0) return 0;
  // the fewest passes digits of 8..9 bits allow, with the narrowest such
  // digit (10-bit digits double the downsweep's per-warp counters and cost
  // occupancy: 200M 30-bit keys took 29 ms in 3 x 10-bit passes against
  // 19 ms in 4 x 8-bit ones; CM_RADIX_MAX_BITS=10 restores them)
#ifndef CM_RADIX_MAX_BITS
#define CM_RADIX_MAX_BITS 9
#endif
  static_assert(CM_RADIX_MAX_BITS <= kRadixBitsMax, "digit wider than the kernels support");
  const int passes_min = (bits + CM_RADIX_MAX_BITS - 1) / CM_RADIX_MAX_BITS;
  const int rb = (bits + passes_min - 1) / passes_min < 8 ? 8 : (bits + passes_min - 1) / passes_min;
  const uint32_t nb = (uint32_t)((n + kSortTile - 1) / kSortTile);
  const uint64_t h = (uint64_t)nb << rb;
  char* p = static_cast<char*>(scratch);
  K* k2 = reinterpret_cast<K*>(p);
  p += n * sizeof(K);
  uint32_t* v2 = reinterpret_cast<uint32_t*>(p);
  p += n * 4;
  uint32_t* hist = reinterpret_cast<uint32_t*>(p);
  p += h * 4;
  uint32_t* part = reinterpret_cast<uint32_t*>(p);
  K* ka = keys;
  uint32_t* va = vals;
  K* kb = k2;
  uint32_t* vb = v2;
  int passes = 0;
// onesweep passes (one histogram kernel + decoupled look-back) measured
// slower than upsweep + scan + downsweep here: 20M-key sort 0.75 -> 0.87 ms
// (the per-digit look-back walks many still-running predecessors)
#ifndef CM_RADIX_ONESWEEP
#define CM_RADIX_ONESWEEP 0
#endif
  const int npass = (bits + rb - 1) / rb;
  if (CM_RADIX_ONESWEEP && n < (1ull << 30) && npass <= 8) {
    // hist: [npass][2^rb] global digit histograms, then digit starts; the
    // look-back status of one pass reuses the per-block histogram area
    uint32_t* ghist = part;
    uint32_t* tctr = ghist + (size_t)npass * (1u << rb);
    uint32_t* status = hist;
    cudaMemsetAsync(ghist, 0, ((size_t)npass * (1u << rb) + npass) * 4, st);
    const unsigned hgrid = (unsigned)std::min<uint64_t>(nb, (uint64_t)sm_count() * 4);
    const size_t hsm = (size_t)npass * kSortWarps * (1u << rb) * 4;
    if (rb == 8) {
      cudaFuncSetAttribute(radix_hist_all<K, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsm);
      radix_hist_all<K, 8><<<hgrid, kSortThreads, hsm, st>>>(ka, n, npass, ghist);
      radix_digit_starts<8><<<npass, kSortThreads, 0, st>>>(ghist);
    } else if (rb == 9) {
      cudaFuncSetAttribute(radix_hist_all<K, 9>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsm);
      radix_hist_all<K, 9><<<hgrid, kSortThreads, hsm, st>>>(ka, n, npass, ghist);
      radix_digit_starts<9><<<npass, kSortThreads, 0, st>>>(ghist);
    } else {
      cudaFuncSetAttribute(radix_hist_all<K, 10>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsm);
      radix_hist_all<K, 10><<<hgrid, kSortThreads, hsm, st>>>(ka, n, npass, ghist);
      radix_digit_starts<10><<<npass, kSortThreads, 0, st>>>(ghist);
    }
    ::cmg::note_launch();
    ::cmg::note_launch();
    for (int ps = 0; ps < npass; ++ps, ++passes) {
      const int shift = ps * rb;
      cudaMemsetAsync(status, 0, ((size_t)nb << rb) * 4, st);
      const uint32_t* ds = ghist + (size_t)ps * (1u << rb);
      if (rb == 8) launch_onesweep<K, 8>(ka, va, kb, vb, n, shift, ds, status, tctr + ps, nb, st);
      else if (rb == 9) launch_onesweep<K, 9>(ka, va, kb, vb, n, shift, ds, status, tctr + ps, nb, st);
      else launch_onesweep<K, 10>(ka, va, kb, vb, n, shift, ds, status, tctr + ps, nb, st);
      K* tk = ka; ka = kb; kb = tk;
      uint32_t* tv = va; va = vb; vb = tv;
    }
    if (ka != keys) {
      cudaMemcpyAsync(keys, ka, n * sizeof(K), cudaMemcpyDeviceToDevice, st);
      cudaMemcpyAsync(vals, va, n * 4, cudaMemcpyDeviceToDevice, st);
    }
    return passes;
  }
  for (int shift = 0; shift < bits; shift += rb, ++passes) {
    if (rb == 8) {
      radix_upsweep<K, 8><<<nb, kSortThreads, 0, st>>>(ka, n, shift, hist, nb); ::cmg::note_launch();
    } else if (rb == 9) {
      radix_upsweep<K, 9><<<nb, kSortThreads, 0, st>>>(ka, n, shift, hist, nb); ::cmg::note_launch();
    } else {
      radix_upsweep<K, 10><<<nb, kSortThreads, 0, st>>>(ka, n, shift, hist, nb); ::cmg::note_launch();
    }
    exclusive_scan<uint32_t, uint32_t>(hist, h, hist, part, 0, st);
    if (rb == 8) launch_downsweep<K, 8>(ka, va, kb, vb, n, shift, hist, nb, st);
    else if (rb == 9) launch_downsweep<K, 9>(ka, va, kb, vb, n, shift, hist, nb, st);
    else launch_downsweep<K, 10>(ka, va, kb, vb, n, shift, hist, nb, st);
    K* tk = ka; ka = kb; kb = tk;
    uint32_t* tv = va; va = vb; vb = tv;
  }
  if (kres && vres) {
    *kres = ka;
    *vres = va;
  } else if (ka != keys) {
    cudaMemcpyAsync(keys, ka, n * sizeof(K), cudaMemcpyDeviceToDevice, st);
    cudaMemcpyAsync(vals, va, n * 4, cudaMemcpyDeviceToDevice, st);
  }
  return passes;
}

}  // namespace cmg
