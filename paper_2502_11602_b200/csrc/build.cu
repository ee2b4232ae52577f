// Index build on sm_100a: K1 bbox -> grid dims -> K2 cell keys -> K3 radix
// sort -> record gather -> K4 unique voxels + flavour tables.
// Replaces Cheesemap::build (map.cpp:22-122).
#include <cmath>
#include <cstring>
#include <string>

#include "index.cuh"
#include "sort_scan.cuh"

namespace cmg {

namespace {

__device__ __forceinline__ unsigned long long ord_of(double d) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(d);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
inline double double_of_ord(unsigned long long u) {
  const unsigned long long b = (u >> 63) ? (u & 0x7fffffffffffffffull) : ~u;
  double d;
  std::memcpy(&d, &b, 8);
  return d;
}

// K1: per-axis min/max (aabb_of_points, geometry.cpp:7-21).
__global__ void bbox_kernel(const double* __restrict__ xyz, uint64_t n,
                            unsigned long long* __restrict__ out /* minx,miny,minz,maxx,maxy,maxz */) {
  double lo[3], hi[3];
  bool any = false;
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < n;
       p += (uint64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double v = xyz[3 * p + a];
      if (!any) {
        lo[a] = hi[a] = v;
      } else {
        lo[a] = (v < lo[a]) ? v : lo[a];
        hi[a] = (hi[a] < v) ? v : hi[a];
      }
    }
    any = true;
  }
  unsigned long long olo[3], ohi[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    olo[a] = any ? ord_of(lo[a]) : ~0ull;
    ohi[a] = any ? ord_of(hi[a]) : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long l2 = __shfl_xor_sync(0xffffffffu, olo[a], o);
      const unsigned long long h2 = __shfl_xor_sync(0xffffffffu, ohi[a], o);
      olo[a] = l2 < olo[a] ? l2 : olo[a];
      ohi[a] = h2 > ohi[a] ? h2 : ohi[a];
    }
  }
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      atomicMin(out + a, olo[a]);
      atomicMax(out + 3 + a, ohi[a]);
    }
  }
}

// K1, 16-byte loads: the cloud as a flat array of 3n doubles read two at a
// time. The launch has a multiple of 3 threads, so the two components a
// thread sees ((2t) mod 3 and the next) stay the same on every stride and
// each thread keeps just two running (min, max) pairs; four loads in
// flight per thread, one set of atomics per block.
__global__ void bbox_flat_kernel(const double2* __restrict__ v2, uint64_t nvec, const double* tail,
                                 unsigned long long* __restrict__ out) {
  const uint64_t T = (uint64_t)gridDim.x * blockDim.x;  // T % 3 == 0
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const int c0 = (int)((2 * t) % 3), c1 = (c0 + 1) % 3;
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);
  double lo0 = kInf, hi0 = -kInf, lo1 = kInf, hi1 = -kInf;
  auto take = [&](const double2 v) {
    lo0 = (v.x < lo0) ? v.x : lo0;
    hi0 = (hi0 < v.x) ? v.x : hi0;
    lo1 = (v.y < lo1) ? v.y : lo1;
    hi1 = (hi1 < v.y) ? v.y : hi1;
  };
  uint64_t e = t;
  for (; e + 3 * T < nvec; e += 4 * T) {
    const double2 a = v2[e], b = v2[e + T], c = v2[e + 2 * T], d = v2[e + 3 * T];
    take(a), take(b), take(c), take(d);
  }
  for (; e < nvec; e += T) take(v2[e]);
  double lo[3], hi[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    lo[a] = c0 == a ? lo0 : (c1 == a ? lo1 : kInf);
    hi[a] = c0 == a ? hi0 : (c1 == a ? hi1 : -kInf);
  }
  if (tail && t == 0) {  // 3n odd: the last z
    const double v = *tail;
    lo[2] = (v < lo[2]) ? v : lo[2];
    hi[2] = (hi[2] < v) ? v : hi[2];
  }
  unsigned long long olo[3], ohi[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    olo[a] = ord_of(lo[a]);
    ohi[a] = ord_of(hi[a]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long l2 = __shfl_xor_sync(0xffffffffu, olo[a], o);
      const unsigned long long h2 = __shfl_xor_sync(0xffffffffu, ohi[a], o);
      olo[a] = l2 < olo[a] ? l2 : olo[a];
      ohi[a] = h2 > ohi[a] ? h2 : ohi[a];
    }
  }
  // one set of six atomics per BLOCK (per warp they are 19 K same-address
  // atomics per axis at 20M points: as long as the reads)
  __shared__ unsigned long long sred[8][6];
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int a = 0; a < 3; ++a) sred[w][a] = olo[a], sred[w][3 + a] = ohi[a];
  }
  __syncthreads();
  if (threadIdx.x < 6) {
    unsigned long long v = sred[0][threadIdx.x];
    for (int x = 1; x < (int)(blockDim.x >> 5); ++x) {
      const unsigned long long u = sred[x][threadIdx.x];
      v = threadIdx.x < 3 ? (u < v ? u : v) : (u > v ? u : v);
    }
    if (threadIdx.x < 3) atomicMin(out + threadIdx.x, v);
    else atomicMax(out + threadIdx.x, v);
  }
}

// K2: key = global_index(voxel_of(p)) (grid.cpp:63-72, grid.hpp:65-67).
template <typename K>
__global__ void keys_kernel(const double* __restrict__ xyz, uint64_t n, DevGrid g,
                            K* __restrict__ keys, uint32_t* __restrict__ vals, uint32_t base = 0) {
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < n;
       p += (uint64_t)gridDim.x * blockDim.x) {
    const double x = xyz[3 * p], y = xyz[3 * p + 1], z = xyz[3 * p + 2];
    const uint64_t i = axis_index(x, g.ox, g.sx, g.nx);
    const uint64_t j = axis_index(y, g.oy, g.sy, g.ny);
    const uint64_t k = g.mode3d ? axis_index(z, g.oz, g.sz, g.nz) : 0;
    keys[p] = (K)(i * (g.ny * g.nz) + j * g.nz + k);
    vals[p] = base + (uint32_t)p;
  }
}

// K2 with 16-byte loads: two consecutive points per thread (48 bytes = three
// aligned double2 loads), both keys and handles stored as one 8-byte word.
template <typename K>
__global__ void keys2_kernel(const double2* __restrict__ v2, uint64_t npairs, DevGrid g,
                             K* __restrict__ keys, uint32_t* __restrict__ vals) {
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < npairs;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const double2 a = v2[3 * t], b = v2[3 * t + 1], c = v2[3 * t + 2];  // x0 y0 | z0 x1 | y1 z1
    const uint64_t i0 = axis_index(a.x, g.ox, g.sx, g.nx);
    const uint64_t j0 = axis_index(a.y, g.oy, g.sy, g.ny);
    const uint64_t k0 = g.mode3d ? axis_index(b.x, g.oz, g.sz, g.nz) : 0;
    const uint64_t i1 = axis_index(b.y, g.ox, g.sx, g.nx);
    const uint64_t j1 = axis_index(c.x, g.oy, g.sy, g.ny);
    const uint64_t k1 = g.mode3d ? axis_index(c.y, g.oz, g.sz, g.nz) : 0;
    const K key0 = (K)(i0 * (g.ny * g.nz) + j0 * g.nz + k0);
    const K key1 = (K)(i1 * (g.ny * g.nz) + j1 * g.nz + k1);
    if constexpr (sizeof(K) == 4) {
      reinterpret_cast<uint2*>(keys)[t] = make_uint2((uint32_t)key0, (uint32_t)key1);
    } else {
      keys[2 * t] = key0;
      keys[2 * t + 1] = key1;
    }
    reinterpret_cast<uint2*>(vals)[t] = make_uint2((uint32_t)(2 * t), (uint32_t)(2 * t + 1));
  }
}

// Sorted order -> 32-byte records; run-start flags for the unique pass.
// Also writes the float records of the filtered predicates (filter.cuh: x, y
// relative to the column corner, z relative to oz) and the handle array.
template <typename K>
__global__ void gather_kernel(const double* __restrict__ xyz, const K* __restrict__ keys,
                              const uint32_t* __restrict__ perm, uint64_t n, DevGrid g,
                              PointRec* __restrict__ rec, FRec* __restrict__ frec,
                              uint32_t* __restrict__ ids, uint32_t* __restrict__ flags) {
  const K nz = (K)g.nz, ny = (K)g.ny;
  // four records per thread per step, every random xyz read in flight first
  constexpr int kG = 4;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t s0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s0 < n; s0 += kG * stride) {
    uint32_t hh[kG];
    double xx[kG], yy[kG], zz[kG];
#pragma unroll
    for (int u = 0; u < kG; ++u) {
      const uint64_t s = s0 + u * stride;
      hh[u] = s < n ? perm[s] : 0u;
    }
#pragma unroll
    for (int u = 0; u < kG; ++u) {
      const uint64_t s = s0 + u * stride;
      if (s < n) {
        xx[u] = xyz[3 * (uint64_t)hh[u]];
        yy[u] = xyz[3 * (uint64_t)hh[u] + 1];
        zz[u] = xyz[3 * (uint64_t)hh[u] + 2];
      }
    }
#pragma unroll
    for (int u = 0; u < kG; ++u) {
    const uint64_t s = s0 + u * stride;
    if (s >= n) break;
    const uint32_t h = hh[u];
    const K key = keys[s];
    double2 a, b;
    a.x = xx[u];
    a.y = yy[u];
    b.x = zz[u];
    const K col = key / nz;
    const uint32_t k = (uint32_t)(key - col * nz);
    uint2 t;
    t.x = h;
    t.y = k;
    b.y = *reinterpret_cast<double*>(&t);
    reinterpret_cast<double2*>(rec + s)[0] = a;
    reinterpret_cast<double2*>(rec + s)[1] = b;
    if (CM_FILTER) {
      const K i = col / ny;
      const K j = col - i * ny;
      FRec f;
      f.x = __double2float_rn(__dsub_rn(a.x, col_corner(g.ox, (uint64_t)i, g.sx)));
      f.y = __double2float_rn(__dsub_rn(a.y, col_corner(g.oy, (uint64_t)j, g.sy)));
      f.z = __double2float_rn(__dsub_rn(b.x, g.oz));
      f.k = k;
      frec[s] = f;
    }
    ids[s] = h;
    if (flags) flags[s] = (s == 0 || keys[s - 1] != keys[s]) ? 1u : 0u;
    }
  }
}

// Per-slice non-empty voxel counts (occupancy_stats, map.cpp:160-165) go
// through a per-block shared-memory histogram when the grid has few slices.
constexpr uint32_t kSliceSmem = 8192;

// Unique voxels in two passes over the sorted keys, no flag / position
// arrays: (1) voxel runs starting in each tile of 4096 keys, (2) after the
// scan of the tile counts, every tile ranks its run starts (blocked: 16
// consecutive keys per thread, one block scan) and writes key, first
// record, z index and the slice counts. 160 MB of key reads at 20M points
// where flags + scan + unique moved 560 MB (0.18 -> ms: see DESIGN.md).
constexpr int kUqThreads = 256;
constexpr int kUqItems = 16;
constexpr int kUqTile = kUqThreads * kUqItems;

template <typename K>
__global__ void __launch_bounds__(kUqThreads) unique_count_kernel(const K* __restrict__ keys,
                                                                  uint64_t n,
                                                                  uint32_t* __restrict__ tile_cnt) {
  __shared__ uint32_t wsum[kUqThreads / 32];
  const uint64_t base = (uint64_t)blockIdx.x * kUqTile;
  uint32_t c = 0;
#pragma unroll
  for (int it = 0; it < kUqItems; ++it) {
    const uint64_t i = base + (uint64_t)it * kUqThreads + threadIdx.x;
    if (i < n) c += (i == 0 || keys[i - 1] != keys[i]) ? 1u : 0u;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t tot = 0;
#pragma unroll
    for (int w = 0; w < kUqThreads / 32; ++w) tot += wsum[w];
    tile_cnt[blockIdx.x] = tot;
  }
}

template <typename K>
__global__ void __launch_bounds__(kUqThreads) unique_write_kernel(
    const K* __restrict__ keys, uint64_t n, const uint32_t* __restrict__ tile_off, uint64_t nz,
    uint64_t* __restrict__ ukey, uint32_t* __restrict__ ustart, uint32_t* __restrict__ uk_k,
    unsigned long long* __restrict__ slice_ne) {
  extern __shared__ uint32_t hist[];  // nz slice counters when they fit, then the warp sums
  const bool local = nz <= kSliceSmem;
  __shared__ uint32_t wsum[kUqThreads / 32];
  if (local)
    for (uint32_t i = threadIdx.x; i < nz; i += blockDim.x) hist[i] = 0;
  const uint64_t b0 = (uint64_t)blockIdx.x * kUqTile + (uint64_t)threadIdx.x * kUqItems;
  K kv[kUqItems];
  K prev = 0;
  bool has_prev = false;
  if (b0 < n && b0 > 0) prev = keys[b0 - 1], has_prev = true;
  uint32_t fl = 0, c = 0;
#pragma unroll
  for (int j = 0; j < kUqItems; ++j) {
    const uint64_t i = b0 + j;
    if (i < n) {
      kv[j] = keys[i];
      const bool f = !has_prev || kv[j] != prev;
      fl |= (uint32_t)f << j;
      c += f;
      prev = kv[j];
      has_prev = true;
    }
  }
  // block exclusive scan of the per-thread counts
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t inc = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += u;
  }
  if (lane == 31) wsum[w] = inc;
  __syncthreads();
  uint32_t woff = 0;
#pragma unroll
  for (int x = 0; x < kUqThreads / 32; ++x) woff += x < w ? wsum[x] : 0u;
  uint32_t u = __ldg(tile_off + blockIdx.x) + woff + inc - c;
#pragma unroll
  for (int j = 0; j < kUqItems; ++j) {
    if ((fl >> j) & 1u) {
      const uint64_t key = (uint64_t)kv[j];
      ukey[u] = key;
      ustart[u] = (uint32_t)(b0 + j);
      const uint32_t k = (uint32_t)(key % nz);
      if (uk_k) uk_k[u] = k;
      if (local) atomicAdd(hist + k, 1u);
      else atomicAdd(slice_ne + k, 1ull);
      ++u;
    }
  }
  if (local) {
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < nz; i += blockDim.x)
      if (hist[i]) atomicAdd(slice_ne + i, (unsigned long long)hist[i]);
  }
}

__global__ void dense_counts_kernel(const uint64_t* __restrict__ ukey,
                                    const uint32_t* __restrict__ ustart, uint64_t U,
                                    uint32_t* __restrict__ cnt) {
  for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < U;
       u += (uint64_t)gridDim.x * blockDim.x)
    cnt[ukey[u]] = ustart[u + 1] - ustart[u];
}

__global__ void hash_insert_kernel(const uint64_t* __restrict__ keys,
                                   const uint32_t* __restrict__ a, const uint32_t* __restrict__ b,
                                   uint64_t m, HashSlot* __restrict__ t, uint64_t mask,
                                   int a_is_index) {
  for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < m;
       u += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t key = keys[u];
    uint64_t s = mix64(key) & mask;
    for (;;) {
      const unsigned long long prev = atomicCAS(
          reinterpret_cast<unsigned long long*>(&t[s].key), (unsigned long long)kEmptyKey,
          (unsigned long long)key);
      if (prev == kEmptyKey) {
        t[s].a = a_is_index ? (uint32_t)u : a[u];
        t[s].b = a_is_index ? 0u : b[u];
        break;
      }
      s = (s + 1) & mask;
    }
  }
}

// Column of each unique voxel; run-start flags over columns.
__global__ void column_flags_kernel(const uint64_t* __restrict__ ukey, uint64_t U, uint64_t nz,
                                    uint32_t* __restrict__ flags) {
  for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < U;
       u += (uint64_t)gridDim.x * blockDim.x)
    flags[u] = (u == 0 || ukey[u - 1] / nz != ukey[u] / nz) ? 1u : 0u;
}

__global__ void column_scatter_kernel(const uint64_t* __restrict__ ukey,
                                      const uint32_t* __restrict__ flags,
                                      const uint32_t* __restrict__ pos, uint64_t U, uint64_t nz,
                                      uint64_t* __restrict__ col_id,
                                      uint32_t* __restrict__ col_vbeg,
                                      uint32_t* __restrict__ col_dense) {
  for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < U;
       u += (uint64_t)gridDim.x * blockDim.x) {
    if (flags[u]) {
      const uint32_t c = pos[u];
      const uint64_t col = ukey[u] / nz;
      col_vbeg[c] = (uint32_t)u;
      if (col_id) col_id[c] = col;
      if (col_dense) col_dense[col] = c;
    }
  }
}

unsigned grid_for(uint64_t n, unsigned threads = 256) {
  const uint64_t want = (n + threads - 1) / threads;
  const uint64_t cap = (uint64_t)sm_count() * 16;
  return (unsigned)std::max<uint64_t>(1, std::min(want, cap));
}

uint64_t next_pow2(uint64_t v) {
  uint64_t p = 1;
  while (p < v) p <<= 1;
  return p;
}

int bit_width(uint64_t v) {
  int b = 0;
  while (v) {
    ++b;
    v >>= 1;
  }
  return b;
}

// grid.cpp:18-27
cm_status axis_dim(double lo, double hi, double cell, uint64_t* out, const char* axis) {
  if (!(cell > 0.0)) {
    set_error(std::string("cell size must be strictly positive (axis ") + axis + ")");
    return CM_INVALID_ARGUMENT;
  }
  const double n = std::floor((hi - lo) / cell) + 1.0;
  if (n >= 9.3e18) {
    set_error("grid axis exceeds the index type capacity");
    return CM_CAPACITY;
  }
  *out = static_cast<uint64_t>(n);
  return CM_OK;
}

struct Events {
  cudaEvent_t e[8];
  int used = 0;
  Events() {
    for (auto& x : e) cudaEventCreate(&x);
  }
  ~Events() {
    for (auto& x : e) cudaEventDestroy(x);
  }
};

template <typename K>
cm_status build_typed(const double* xyz, uint64_t n, cudaStream_t st, cm_index* ix,
                      Events& ev) {
  const DevGrid& g = ix->g;
  K* keys = nullptr;
  uint32_t* perm = nullptr;
  void* scratch = nullptr;
  CM_CUDA_TRY(dev_alloc_t(&keys, n, st));
  CM_CUDA_TRY(dev_alloc_t(&perm, n, st));
  CM_CUDA_TRY(dev_alloc(&scratch, radix_scratch_bytes<K>(n), st));
  if ((reinterpret_cast<uintptr_t>(xyz) & 15u) == 0 && n >= 2) {
    const uint64_t npairs = n / 2;
    keys2_kernel<K><<<grid_for(npairs), 256, 0, st>>>(reinterpret_cast<const double2*>(xyz), npairs, g,
                                                     keys, perm);
    ::cmg::note_launch();
    if (n & 1) {  // the last point
      keys_kernel<K><<<1, 32, 0, st>>>(xyz + 3 * (n - 1), 1, g, keys + (n - 1), perm + (n - 1),
                                       (uint32_t)(n - 1));
      ::cmg::note_launch();
    }
  } else {
    keys_kernel<K><<<grid_for(n), 256, 0, st>>>(xyz, n, g, keys, perm); ::cmg::note_launch();
  }
  cudaEventRecord(ev.e[2], st);
  ix->key_bits = bit_width(ix->V - 1);
  // the sorted pairs stay where the last pass left them (no copy back)
  K* skeys = keys;
  uint32_t* sperm = perm;
  ix->timing.sort_passes =
      (uint32_t)radix_sort_pairs<K>(keys, perm, n, ix->key_bits, scratch, st, &skeys, &sperm);
  cudaEventRecord(ev.e[3], st);

  CM_CUDA_TRY(dev_alloc_t(&ix->rec, n, st));
  if (CM_FILTER) CM_CUDA_TRY(dev_alloc_t(&ix->frec, n, st));
  CM_CUDA_TRY(dev_alloc_t(&ix->ids, n, st));
  uint32_t* flags = nullptr;
  uint32_t* pos = nullptr;
  uint32_t* part = nullptr;
  CM_CUDA_TRY(dev_alloc_t(&flags, n, st));
  CM_CUDA_TRY(dev_alloc_t(&pos, n + 1, st));
  CM_CUDA_TRY(dev_alloc_t(&part, scan_part_elems(n), st));
  gather_kernel<K><<<grid_for(n), 256, 0, st>>>(xyz, skeys, sperm, n, g, ix->rec, ix->frec, ix->ids, nullptr); ::cmg::note_launch();
  cudaEventRecord(ev.e[4], st);
  // voxel runs per tile -> tile offsets (pos[0 .. ntiles], total at the end)
  const uint64_t ntiles = (n + kUqTile - 1) / kUqTile;
  unique_count_kernel<K><<<(unsigned)ntiles, kUqThreads, 0, st>>>(skeys, n, flags); ::cmg::note_launch();
  exclusive_scan<uint32_t, uint32_t>(flags, ntiles, pos, part, 1, st);
  uint32_t U32 = 0;
  CM_CUDA_TRY(cudaMemcpyAsync(&U32, pos + ntiles, 4, cudaMemcpyDeviceToHost, st));
  CM_CUDA_TRY(cudaStreamSynchronize(st));
  const uint64_t U = U32;
  ix->U = U;
  const int flavor = ix->opts.flavor;
  unsigned long long* slice_ne = nullptr;
  CM_CUDA_TRY(dev_alloc_t(&ix->ukey, U, st));
  CM_CUDA_TRY(dev_alloc_t(&ix->ustart, U + 1, st));
  if (flavor == CM_MIXED) CM_CUDA_TRY(dev_alloc_t(&ix->uk_k, U, st));
  CM_CUDA_TRY(dev_alloc_t(&slice_ne, g.nz, st));
  CM_CUDA_TRY(cudaMemsetAsync(slice_ne, 0, g.nz * 8, st));
  const uint32_t n32 = (uint32_t)n;
  CM_CUDA_TRY(cudaMemcpyAsync(ix->ustart + U, &n32, 4, cudaMemcpyHostToDevice, st));
  const size_t hsmem = g.nz <= kSliceSmem ? g.nz * 4 : 0;
  unique_write_kernel<K><<<(unsigned)ntiles, kUqThreads, hsmem, st>>>(skeys, n, pos, g.nz, ix->ukey,
                                                                     ix->ustart, ix->uk_k, slice_ne);
  ::cmg::note_launch();
  ix->slice_ne.assign(g.nz, 0);
  CM_CUDA_TRY(cudaMemcpyAsync(ix->slice_ne.data(), slice_ne, g.nz * 8, cudaMemcpyDeviceToHost, st));
  dev_free(keys, st);
  dev_free(perm, st);
  dev_free(scratch, st);

  if (flavor == CM_DENSE) {
    CM_CUDA_TRY(dev_alloc_t(&ix->dense_off, ix->V + 1, st));
    CM_CUDA_TRY(cudaMemsetAsync(ix->dense_off, 0, (ix->V + 1) * 4, st));
    dense_counts_kernel<<<grid_for(U), 256, 0, st>>>(ix->ukey, ix->ustart, U, ix->dense_off); ::cmg::note_launch();
    uint32_t* vpart = nullptr;
    CM_CUDA_TRY(dev_alloc_t(&vpart, scan_part_elems(ix->V), st));
    exclusive_scan<uint32_t, uint32_t>(ix->dense_off, ix->V, ix->dense_off, vpart, 1, st);
    dev_free(vpart, st);
  } else if (flavor == CM_SPARSE) {
    const uint64_t cap = next_pow2(std::max<uint64_t>(2 * U, 1024));
    ix->vmask = cap - 1;
    CM_CUDA_TRY(dev_alloc_t(&ix->vhash, cap, st));
    CM_CUDA_TRY(cudaMemsetAsync(ix->vhash, 0xff, cap * sizeof(HashSlot), st));
    hash_insert_kernel<<<grid_for(U), 256, 0, st>>>(ix->ukey, ix->ustart, ix->ustart + 1, U,
                                                    ix->vhash, ix->vmask, 0); ::cmg::note_launch();
  } else {
    // mixed: 2D column table over the (i, j) footprint + sparse z lists
    column_flags_kernel<<<grid_for(U), 256, 0, st>>>(ix->ukey, U, g.nz, flags); ::cmg::note_launch();
    exclusive_scan<uint32_t, uint32_t>(flags, U, pos, part, 1, st);
    uint32_t C32 = 0;
    CM_CUDA_TRY(cudaMemcpyAsync(&C32, pos + U, 4, cudaMemcpyDeviceToHost, st));
    CM_CUDA_TRY(cudaStreamSynchronize(st));
    const uint64_t C = C32;
    ix->C = C;
    const uint64_t footprint = g.nx * g.ny;
    CM_CUDA_TRY(dev_alloc_t(&ix->col_vbeg, C + 1, st));
    const uint32_t U32v = (uint32_t)U;
    CM_CUDA_TRY(cudaMemcpyAsync(ix->col_vbeg + C, &U32v, 4, cudaMemcpyHostToDevice, st));
    // The column table densifies by the reference's rule for a mixed slice
    // (map.cpp:106-108), applied to the 2D footprint.
    const bool dense_fp =
        static_cast<double>(C) / static_cast<double>(footprint) >= ix->opts.densify_threshold;
    uint64_t* col_id = nullptr;
    if (dense_fp) {
      CM_CUDA_TRY(dev_alloc_t(&ix->col_dense, footprint, st));
      CM_CUDA_TRY(cudaMemsetAsync(ix->col_dense, 0xff, footprint * 4, st));
    } else {
      CM_CUDA_TRY(dev_alloc_t(&col_id, C, st));
    }
    column_scatter_kernel<<<grid_for(U), 256, 0, st>>>(ix->ukey, flags, pos, U, g.nz, col_id,
                                                       ix->col_vbeg, ix->col_dense); ::cmg::note_launch();
    if (!dense_fp) {
      const uint64_t cap = next_pow2(std::max<uint64_t>(2 * C, 1024));
      ix->cmask = cap - 1;
      CM_CUDA_TRY(dev_alloc_t(&ix->chash, cap, st));
      CM_CUDA_TRY(cudaMemsetAsync(ix->chash, 0xff, cap * sizeof(HashSlot), st));
      hash_insert_kernel<<<grid_for(C), 256, 0, st>>>(col_id, nullptr, nullptr, C, ix->chash,
                                                      ix->cmask, 1); ::cmg::note_launch();
      dev_free(col_id, st);
    }
  }
  dev_free(flags, st);
  dev_free(pos, st);
  dev_free(part, st);
  dev_free(slice_ne, st);
  CM_CUDA_TRY(cudaGetLastError());
  return CM_OK;
}

}  // namespace

// aabb_of_points (geometry.cpp:7-21) of n device points -> host lo / hi
// (+inf / -inf for n = 0). Synchronous; `after` (optional) is recorded once
// the reduction is queued.
cm_status bbox_dev(const double* xyz, uint64_t n, cudaStream_t st, double lo[3], double hi[3],
                   cudaEvent_t after) {
  unsigned long long* bb = nullptr;
  CM_CUDA_TRY(dev_alloc_t(&bb, 6, st));
  unsigned long long init[6] = {~0ull, ~0ull, ~0ull, 0ull, 0ull, 0ull};
  CM_CUDA_TRY(cudaMemcpyAsync(bb, init, sizeof(init), cudaMemcpyHostToDevice, st));
  if (n) {
    if ((reinterpret_cast<uintptr_t>(xyz) & 15u) == 0 && n >= 4096) {
      const uint64_t nvec = 3 * n / 2;
      unsigned grid = grid_for(nvec);
      grid = std::max(3u, grid - grid % 3u);  // a multiple of 3 threads in all
      bbox_flat_kernel<<<grid, 256, 0, st>>>(reinterpret_cast<const double2*>(xyz), nvec,
                                             (3 * n) & 1 ? xyz + 3 * n - 1 : nullptr, bb);
    } else {
      bbox_kernel<<<grid_for(n), 256, 0, st>>>(xyz, n, bb);
    }
    ::cmg::note_launch();
    CM_CUDA_TRY(cudaGetLastError());
  }
  unsigned long long hb[6];
  CM_CUDA_TRY(cudaMemcpyAsync(hb, bb, sizeof(hb), cudaMemcpyDeviceToHost, st));
  if (after) cudaEventRecord(after, st);
  CM_CUDA_TRY(cudaStreamSynchronize(st));
  dev_free(bb, st);
  for (int a = 0; a < 3; ++a) {
    lo[a] = n ? double_of_ord(hb[a]) : __builtin_inf();
    hi[a] = n ? double_of_ord(hb[3 + a]) : -__builtin_inf();
  }
  return CM_OK;
}

cm_status build_index(const double* xyz, uint64_t n, const cm_build_options& o, cudaStream_t st,
                      cm_index* ix, const double* bounds6) {
  // Check order follows map.cpp:23-39.
  if (n == 0) {
    set_error("point cloud is empty");
    return CM_EMPTY_CLOUD;
  }
  if (!(o.densify_threshold > 0.0) || o.densify_threshold > 1.0) {
    set_error("densify threshold must be in (0, 1]");
    return CM_INVALID_ARGUMENT;
  }
  if (o.flavor < CM_DENSE || o.flavor > CM_MIXED || (o.mode != CM_TWOD && o.mode != CM_THREED)) {
    set_error("unknown flavor or grid mode");
    return CM_INVALID_ARGUMENT;
  }
  if (n >= (1ull << 32)) {
    set_error("clouds of 2^32 points or more exceed the device handle type (u32)");
    return CM_CAPACITY;
  }
  ix->opts = o;
  ix->n = n;
  Events ev;
  cudaEventRecord(ev.e[0], st);
  double lo[3], hi[3];
  {
    cm_status bs = bbox_dev(xyz, n, st, lo, hi, ev.e[1]);
    if (bs != CM_OK) return bs;
  }
  if (bounds6) {
    // An explicit (e.g. global, all-reduced) bounding box: every point must
    // lie inside it, as voxel_of demands (grid.cpp:64-66).
    for (int a = 0; a < 3; ++a) {
      if (!(lo[a] >= bounds6[a] && hi[a] <= bounds6[3 + a])) {
        set_error("point lies outside the grid bounding box");
        return CM_OUT_OF_DOMAIN;
      }
      lo[a] = bounds6[a];
      hi[a] = bounds6[3 + a];
    }
  }
  // grid_dims (grid.cpp:41-61)
  DevGrid& g = ix->g;
  g.ox = lo[0], g.oy = lo[1], g.oz = lo[2];
  g.bx0 = lo[0], g.by0 = lo[1], g.bz0 = lo[2];
  g.bx1 = hi[0], g.by1 = hi[1], g.bz1 = hi[2];
  g.sx = o.cell_x, g.sy = o.cell_y, g.sz = o.cell_z;
  g.mode3d = o.mode == CM_THREED;
  cm_status s;
  if ((s = axis_dim(lo[0], hi[0], o.cell_x, &g.nx, "x")) != CM_OK) return s;
  if ((s = axis_dim(lo[1], hi[1], o.cell_y, &g.ny, "y")) != CM_OK) return s;
  if (g.mode3d) {
    if ((s = axis_dim(lo[2], hi[2], o.cell_z, &g.nz, "z")) != CM_OK) return s;
  } else {
    g.nz = 1;
  }
  const uint64_t limit = 1ull << 63;
  if ((g.ny != 0 && g.nx > limit / g.ny) || (g.nz != 0 && g.nx * g.ny > limit / g.nz)) {
    set_error("voxel count overflows the index type");
    return CM_CAPACITY;
  }
  ix->V = g.nx * g.ny * g.nz;
  if (o.flavor == CM_DENSE && ix->V > o.dense_voxel_cap) {  // map.cpp:35-39
    set_error("dense grid of " + std::to_string(ix->V) +
              " voxels exceeds the cap; use the sparse or mixed flavor");
    return CM_CAPACITY;
  }
  if (o.flavor == CM_DENSE && ix->V >= (1ull << 32) - 1) {
    set_error("dense offset table needs V + 1 < 2^32 entries on the device");
    return CM_CAPACITY;
  }
  s = ix->V <= (1ull << 32) ? build_typed<uint32_t>(xyz, n, st, ix, ev)
                            : build_typed<uint64_t>(xyz, n, st, ix, ev);
  if (s != CM_OK) return s;
  cudaEventRecord(ev.e[5], st);
  CM_CUDA_TRY(cudaStreamSynchronize(st));
  float ms;
  cudaEventElapsedTime(&ms, ev.e[0], ev.e[5]);
  ix->timing.total_ms = ms;
  cudaEventElapsedTime(&ms, ev.e[0], ev.e[1]);
  ix->timing.bbox_ms = ms;
  cudaEventElapsedTime(&ms, ev.e[1], ev.e[2]);
  ix->timing.keys_ms = ms;
  cudaEventElapsedTime(&ms, ev.e[2], ev.e[3]);
  ix->timing.sort_ms = ms;
  cudaEventElapsedTime(&ms, ev.e[3], ev.e[4]);
  ix->timing.gather_ms = ms;
  cudaEventElapsedTime(&ms, ev.e[4], ev.e[5]);
  ix->timing.tables_ms = ms;
  return CM_OK;
}

}  // namespace cmg
