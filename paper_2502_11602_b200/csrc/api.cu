// C ABI (include/cmgpu.h): argument checks, host/device staging, ownership.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <random>
#include <string>
#include <vector>

#include "index.cuh"
#include "sort_scan.cuh"

namespace cmg {

namespace {
thread_local std::string g_last_error;
std::mutex g_pool_mu;
}  // namespace

void set_error(const std::string& msg) { g_last_error = msg; }

static std::atomic<uint64_t> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int sm_count() {
  static int cached[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cached[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = v > 0 ? v : 1;
  }
  return cached[dev];
}

// The library's device memory comes from a PRIVATE stream-ordered pool per
// device (not the device's default pool), so torch or any other user of the
// default pool is unaffected by what this pool caches. Defaults are
// conservative: nothing is reserved up front, the pool grows with demand in
// large blocks (dev_alloc), and at most 1/8 of HBM stays cached across
// synchronisations. Serving processes that own the GPU opt in
// to more with cm_pool_configure (the bench does: a reservation carved into
// later requests avoids mapping fresh memory inside a call — measured 0.3-12
// ms per cudaMallocAsync once the pool's chunks fragment) or with
// CMGPU_POOL_KEEP_FRAC / CMGPU_POOL_RESERVE_GB in the environment.
struct DevicePool {
  cudaMemPool_t pool = nullptr;
  bool tried = false;
};
DevicePool g_pools[kMaxDevices];

static cudaError_t reserve_in_pool(cudaMemPool_t pool, uint64_t bytes) {
  if (!bytes) return cudaSuccess;
  void* p = nullptr;
  cudaError_t e = cudaMallocFromPoolAsync(&p, bytes, pool, 0);
  if (e == cudaSuccess) cudaFreeAsync(p, 0);
  cudaStreamSynchronize(0);
  cudaGetLastError();
  return e;
}

static cudaMemPool_t device_pool(int dev) {
  if (dev < 0 || dev >= kMaxDevices) return nullptr;
  std::lock_guard<std::mutex> lk(g_pool_mu);
  DevicePool& dp = g_pools[dev];
  if (!dp.tried) {
    dp.tried = true;
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    if (cudaMemPoolCreate(&dp.pool, &props) != cudaSuccess) {
      cudaGetLastError();
      dp.pool = nullptr;
      return nullptr;
    }
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    double keep = 0.125;
    if (const char* kf = std::getenv("CMGPU_POOL_KEEP_FRAC")) keep = std::atof(kf);
    uint64_t thr = (uint64_t)((double)tot * std::min(1.0, std::max(0.0, keep)));
    cudaMemPoolSetAttribute(dp.pool, cudaMemPoolAttrReleaseThreshold, &thr);
    if (const char* r = std::getenv("CMGPU_POOL_RESERVE_GB"))
      reserve_in_pool(dp.pool, (uint64_t)(std::atof(r) * (double)(1ull << 30)));
  }
  return dp.pool;
}

cudaError_t dev_alloc(void** p, size_t bytes, cudaStream_t st) {
  int dev = 0;
  cudaGetDevice(&dev);
  cudaMemPool_t pool = device_pool(dev);
  auto alloc = [&]() {
    return pool ? cudaMallocFromPoolAsync(p, bytes == 0 ? 16 : bytes, pool, st)
                : cudaMallocAsync(p, bytes == 0 ? 16 : bytes, st);
  };
  // Growth on demand, geometric and in one block: when a large request
  // exceeds what the pool holds free, the pool first takes one block of
  // four times the request (at least what it already holds), so this and the
  // next requests carve from a few large blocks instead of mapping a fresh
  // one per call. Without it the host-buffer search of config 1 took 79-139
  // ms per 20M-query call (the pool mapping memory inside the calls: 11.7 GB
  // reserved, fragmented) against 72 ms with one up-front reservation; with
  // it the second call onward takes 72 ms (the first one maps the blocks:
  // 0.3 s once). Factor 2 left it at 80 ms. The pool never grows this way
  // past its release threshold (it would be trimmed at the next
  // synchronisation) nor past half of the free memory, and small workloads
  // (requests under 64 MB) never trigger it. CMGPU_POOL_GROW=f sets the
  // factor, 0 turns it off.
  static const bool grow_on = !(std::getenv("CMGPU_POOL_GROW") && std::atof(std::getenv("CMGPU_POOL_GROW")) == 0.0);
  if (pool && grow_on && bytes >= (64ull << 20)) {
    uint64_t reserved = 0, used = 0, thr = 0;
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    if (reserved - std::min(reserved, used) < bytes) {
      size_t fr = 0, tot = 0;
      cudaMemGetInfo(&fr, &tot);
      static const double gf = std::getenv("CMGPU_POOL_GROW") ? std::max(1.0, std::atof(std::getenv("CMGPU_POOL_GROW"))) : 4.0;
      uint64_t grow = std::max<uint64_t>((uint64_t)(gf * (double)bytes), (uint64_t)((double)reserved * gf / 4.0));
      grow = std::min<uint64_t>(grow, (uint64_t)fr / 2);
      if (thr > reserved) grow = std::min<uint64_t>(grow, thr - reserved); else grow = 0;
      if (grow >= bytes) {
        void* blk = nullptr;
        if (cudaMallocFromPoolAsync(&blk, grow, pool, st) == cudaSuccess) cudaFreeAsync(blk, st);
        else cudaGetLastError();
      }
    }
  }
  cudaError_t e = alloc();
  if (e == cudaErrorMemoryAllocation) {
    // the pool keeps freed blocks cached: give them back to the device and
    // retry once
    cudaGetLastError();
    cudaDeviceSynchronize();
    if (pool) cudaMemPoolTrimTo(pool, 0);
    e = alloc();
  }
  return e;
}

void dev_free(void* p, cudaStream_t st) {
  if (p) cudaFreeAsync(p, st);
}

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

cm_status stage_input(const void* p, size_t bytes, cudaStream_t st, InBuf* out) {
  out->st = st;
  if (is_device_ptr(p) || bytes == 0) {
    out->dev = p;
    return CM_OK;
  }
  CM_CUDA_TRY(dev_alloc(&out->owned, bytes, st));
  CM_CUDA_TRY(cudaMemcpyAsync(out->owned, p, bytes, cudaMemcpyHostToDevice, st));
  out->dev = out->owned;
  return CM_OK;
}

}  // namespace cmg

struct cm_csr {
  uint64_t nq = 0, nnz = 0;
  uint64_t* row_ptr = nullptr;
  uint32_t* cols = nullptr;
  int device = 0;
};

using namespace cmg;

namespace {

// An output the kernels write: the caller's device pointer, or a device
// buffer copied back to the caller's host pointer on finish().
template <typename T>
struct OutBuf {
  T* user = nullptr;
  T* dev = nullptr;
  bool owned = false;
  size_t count = 0;
  cudaStream_t st = nullptr;
  cm_status init(T* p, size_t n, cudaStream_t s) {
    user = p, count = n, st = s;
    if (!p) return CM_OK;
    if (is_device_ptr(p)) {
      dev = p;
      return CM_OK;
    }
    owned = true;
    CM_CUDA_TRY(dev_alloc_t(&dev, n, s));
    return CM_OK;
  }
  cm_status finish() {
    if (owned && count) CM_CUDA_TRY(cudaMemcpyAsync(user, dev, count * sizeof(T), cudaMemcpyDeviceToHost, st));
    return CM_OK;
  }
  bool host() const { return owned; }
  ~OutBuf() {
    if (owned) dev_free(dev, st);
  }
};

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

cm_status check_index(const cm_index* ix) {
  if (!ix) {
    set_error("null index");
    return CM_INVALID_ARGUMENT;
  }
  return CM_OK;
}

cm_status check_kernel(int kernel) {
  if (kernel != CM_SPHERE && kernel != CM_CUBE && kernel != CM_CYLINDER) {
    set_error("unknown kernel (CM_SPHERE = 0, CM_CUBE = 1, CM_CYLINDER = 2)");
    return CM_INVALID_ARGUMENT;
  }
  return CM_OK;
}

cm_status sync_if(bool host, cudaStream_t st) {
  if (host) CM_CUDA_TRY(cudaStreamSynchronize(st));
  return CM_OK;
}

#define CM_TRY(expr)                 \
  do {                               \
    cm_status _s = (expr);           \
    if (_s != CM_OK) return _s;      \
  } while (0)

}  // namespace

extern "C" {

void cm_default_options(cm_build_options* o) {
  o->flavor = CM_DENSE;
  o->mode = CM_THREED;
  o->cell_x = o->cell_y = o->cell_z = 1.0;
  o->reorder = 0;
  o->densify_threshold = 0.80;
  o->dense_voxel_cap = 1ull << 32;
}

const char* cm_last_error(void) { return g_last_error.c_str(); }

uint64_t cm_launch_count(void) { return g_launches.load(); }

cm_status cm_debug_query_stats(uint64_t* out8, int reset) {
  if (!out8) return CM_INVALID_ARGUMENT;
  query_stats(out8, reset);
  return CM_OK;
}

cm_status cm_debug_pool_bytes(int device, int trim, uint64_t* reserved, uint64_t* used) {
  if (!reserved || !used) {
    set_error("null output pointer");
    return CM_INVALID_ARGUMENT;
  }
  DeviceGuard dg(device);
  cudaMemPool_t pool = device_pool(device);
  if (!pool) {
    set_error("no device pool");
    return CM_CUDA;
  }
  if (trim) {
    CM_CUDA_TRY(cudaDeviceSynchronize());
    CM_CUDA_TRY(cudaMemPoolTrimTo(pool, 0));
  }
  uint64_t r = 0, u = 0;  // the attributes are cuuint64_t (64-bit)
  CM_CUDA_TRY(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &r));
  CM_CUDA_TRY(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &u));
  *reserved = r;
  *used = u;
  return CM_OK;
}

cm_status cm_pool_configure(int device, uint64_t keep_bytes, uint64_t reserve_bytes) {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
    cudaGetLastError();
    set_error("device ordinal out of range");
    return CM_INVALID_ARGUMENT;
  }
  DeviceGuard dg(device);
  cudaMemPool_t pool = device_pool(device);
  if (!pool) {
    set_error("no device pool");
    return CM_CUDA;
  }
  CM_CUDA_TRY(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep_bytes));
  if (reserve_in_pool(pool, reserve_bytes) != cudaSuccess) {
    set_error("pool reservation failed");
    return CM_CUDA;
  }
  return CM_OK;
}

const char* cm_status_name(cm_status s) {
  switch (s) {
    case CM_OK: return "CM_OK";
    case CM_PARSE: return "CM_PARSE";
    case CM_IO: return "CM_IO";
    case CM_EMPTY_CLOUD: return "CM_EMPTY_CLOUD";
    case CM_INVALID_ARGUMENT: return "CM_INVALID_ARGUMENT";
    case CM_CAPACITY: return "CM_CAPACITY";
    case CM_OUT_OF_DOMAIN: return "CM_OUT_OF_DOMAIN";
    case CM_CUDA: return "CM_CUDA";
    case CM_NCCL: return "CM_NCCL";
  }
  return "CM_UNKNOWN";
}

static cm_status build_common(const double* xyz, uint64_t n, const cm_build_options* opts,
                               const double* bounds6, int device, void* stream, cm_index** out) {
  if (!out) {
    set_error("null output handle");
    return CM_INVALID_ARGUMENT;
  }
  *out = nullptr;
  cm_build_options o;
  if (opts) o = *opts;
  else cm_default_options(&o);
  if (n == 0) {
    set_error("point cloud is empty");
    return CM_EMPTY_CLOUD;
  }
  if (!xyz) {
    set_error("null point pointer");
    return CM_INVALID_ARGUMENT;
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    set_error("no CUDA device available");
    return CM_CUDA;
  }
  if (device < 0 || device >= ndev) {
    set_error("device ordinal out of range");
    return CM_INVALID_ARGUMENT;
  }
  DeviceGuard dg(device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cm_index* ix = new cm_index();
  ix->device = device;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, st);
  InBuf in;
  cm_status s = stage_input(xyz, n * 3 * sizeof(double), st, &in);
  cudaEventRecord(e1, st);
  if (s == CM_OK) s = build_index(static_cast<const double*>(in.dev), n, o, st, ix, bounds6);
  float h2d = 0;
  if (s == CM_OK) {
    cudaEventElapsedTime(&h2d, e0, e1);
    ix->timing.h2d_ms = in.owned ? h2d : 0.0;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (s != CM_OK) {
    cudaStreamSynchronize(st);
    cm_free(ix);
    return s;
  }
  *out = ix;
  return CM_OK;
}

cm_status cm_build(const double* xyz, uint64_t n, const cm_build_options* opts, int device,
                   void* stream, cm_index** out) {
  return build_common(xyz, n, opts, nullptr, device, stream, out);
}

cm_status cm_build_in_bounds(const double* xyz, uint64_t n, const cm_build_options* opts,
                             const double* bounds_min, const double* bounds_max, int device,
                             void* stream, cm_index** out) {
  if (!bounds_min || !bounds_max) {
    set_error("null bounds");
    return CM_INVALID_ARGUMENT;
  }
  const double b6[6] = {bounds_min[0], bounds_min[1], bounds_min[2],
                        bounds_max[0], bounds_max[1], bounds_max[2]};
  return build_common(xyz, n, opts, b6, device, stream, out);
}

cm_status cm_free(cm_index* ix) {
  if (!ix) return CM_OK;
  DeviceGuard dg(ix->device);
  cudaDeviceSynchronize();
  void* ptrs[] = {ix->rec,   ix->ukey,      ix->ustart, ix->uk_k,     ix->dense_off,
                  ix->vhash, ix->col_dense, ix->chash,  ix->col_vbeg, ix->rec_of,
                  ix->frec,  ix->ids};
  for (void* p : ptrs)
    if (p) cudaFreeAsync(p, 0);
  cudaStreamSynchronize(0);
  delete ix;
  return CM_OK;
}

uint64_t cm_size(const cm_index* ix) { return ix ? ix->n : 0; }

cm_status cm_get_grid(const cm_index* ix, cm_grid_params* o) {
  CM_TRY(check_index(ix));
  const DevGrid& g = ix->g;
  o->origin[0] = g.ox, o->origin[1] = g.oy, o->origin[2] = g.oz;
  o->cell[0] = g.sx, o->cell[1] = g.sy, o->cell[2] = g.sz;
  o->nx = g.nx, o->ny = g.ny, o->nz = g.nz;
  o->mode = g.mode3d ? CM_THREED : CM_TWOD;
  o->bounds_min[0] = g.bx0, o->bounds_min[1] = g.by0, o->bounds_min[2] = g.bz0;
  o->bounds_max[0] = g.bx1, o->bounds_max[1] = g.by1, o->bounds_max[2] = g.bz1;
  return CM_OK;
}

// occupancy_stats (map.cpp:150-171); slice flags by map.cpp:106-108.
cm_status cm_get_occupancy(const cm_index* ix, cm_occupancy* o, uint8_t* slice_dense,
                           uint64_t* slice_non_empty, uint64_t cap) {
  CM_TRY(check_index(ix));
  o->total_voxels = ix->V;
  o->non_empty = ix->U;
  o->empty_fraction = static_cast<double>(ix->V - ix->U) / static_cast<double>(ix->V);
  o->n_slices = ix->slice_ne.size();
  o->n_columns = ix->C;
  const double footprint = static_cast<double>(ix->g.nx * ix->g.ny);
  for (uint64_t k = 0; k < ix->slice_ne.size() && k < cap; ++k) {
    if (slice_non_empty) slice_non_empty[k] = ix->slice_ne[k];
    if (slice_dense)
      slice_dense[k] = static_cast<double>(ix->slice_ne[k]) / footprint >= ix->opts.densify_threshold;
  }
  return CM_OK;
}

cm_status cm_get_memory_report(const cm_index* ix, cm_memory_report* r) {
  CM_TRY(check_index(ix));
  if (!r) {
    set_error("null output pointer");
    return CM_INVALID_ARGUMENT;
  }
  // the reference's cost model (map.cpp:14-18)
  constexpr uint64_t kHandleBytes = 8, kDenseSlotBytes = 8, kSparseEntryBytes = 64,
                     kMixedDenseCellBytes = 24, kSliceHeaderBytes = 48;
  *r = cm_memory_report{};
  r->handle_bytes = kHandleBytes * ix->n;
  if (ix->opts.flavor == CM_DENSE) {
    r->structure_bytes = kDenseSlotBytes * (ix->V + 1);
  } else if (ix->opts.flavor == CM_SPARSE) {
    r->structure_bytes = kSparseEntryBytes * ix->U;
  } else {
    const uint64_t footprint = ix->g.nx * ix->g.ny;
    for (const uint64_t ne : ix->slice_ne) {
      const bool dense = static_cast<double>(ne) / static_cast<double>(footprint) >=
                         ix->opts.densify_threshold;
      r->structure_bytes += kSliceHeaderBytes + (dense ? kMixedDenseCellBytes * footprint
                                                       : kSparseEntryBytes * ne);
    }
  }
  r->total_bytes = r->handle_bytes + r->structure_bytes;
  // this index's own HBM (cm_index, index.cuh)
  uint64_t d = sizeof(PointRec) * ix->n;
  if (ix->ukey) d += 8 * ix->U;
  if (ix->ustart) d += 4 * (ix->U + 1);
  if (ix->uk_k) d += 4 * ix->U;
  if (ix->dense_off) d += 4 * (ix->V + 1);
  if (ix->vhash) d += sizeof(HashSlot) * (ix->vmask + 1);
  if (ix->col_dense) d += 4 * ix->g.nx * ix->g.ny;
  if (ix->chash) d += sizeof(HashSlot) * (ix->cmask + 1);
  if (ix->col_vbeg) d += 4 * (ix->C + 1);
  r->device_bytes = d;
  return CM_OK;
}

cm_status cm_get_build_timing(const cm_index* ix, cm_build_timing* o) {
  CM_TRY(check_index(ix));
  *o = ix->timing;
  return CM_OK;
}

}  // extern "C"

namespace cmg {
namespace apik {
__global__ void export_kernel(const PointRec* __restrict__ rec, uint64_t n, DevGrid g,
                              uint64_t* __restrict__ keys, uint32_t* __restrict__ ids) {
  for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < n;
       s += (uint64_t)gridDim.x * blockDim.x) {
    const PointRec r = rec[s];
    if (ids) ids[s] = r.id;
    if (keys) {
      const uint64_t i = axis_index(r.x, g.ox, g.sx, g.nx);
      const uint64_t j = axis_index(r.y, g.oy, g.sy, g.ny);
      keys[s] = i * (g.ny * g.nz) + j * g.nz + r.k;
    }
  }
}

// Test hook: drop the first record of the first non-empty voxel from the
// tables (map.cpp:194-223 drops one stored handle): every voxel span at or
// below that voxel starts one record later.
// Removes one stored point from every query's view (its x becomes NaN, so
// no kernel predicate accepts it) — the effect of the reference's hook,
// which pops a handle out of a voxel list (map.cpp:194-223). The point is
// the middle one in cell order, reachable from most query centres.
__global__ void corrupt_kernel(PointRec* rec, FRec* frec, uint64_t at) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    rec[at].x = __longlong_as_double(0x7ff8000000000000ll);
    if (frec) frec[at].x = __int_as_float(0x7fc00000);
  }
}
__global__ void add_offset_kernel(uint64_t* v, uint64_t n, uint64_t off) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    v[i] += off;
}
}  // namespace apik
}  // namespace cmg

extern "C" {

cm_status cm_export_voxels(const cm_index* ix, uint64_t* keys, uint32_t* handles) {
  CM_TRY(check_index(ix));
  DeviceGuard dg(ix->device);
  cudaStream_t st = 0;
  OutBuf<uint64_t> k;
  OutBuf<uint32_t> h;
  CM_TRY(k.init(keys, ix->n, st));
  CM_TRY(h.init(handles, ix->n, st));
  apik::export_kernel<<<(unsigned)std::min<uint64_t>((ix->n + 255) / 256, 4096), 256, 0, st>>>(
      ix->rec, ix->n, ix->g, k.dev, h.dev); ::cmg::note_launch();
  CM_CUDA_TRY(cudaGetLastError());
  CM_TRY(k.finish());
  CM_TRY(h.finish());
  CM_CUDA_TRY(cudaStreamSynchronize(st));
  return CM_OK;
}

}  // extern "C"

namespace cmg {
namespace apik {
// The span [b, e) of voxel (i, j, k) in the cell-ordered records, and the
// handles stored there (ascending, as the reference stores a voxel's points
// in cloud order, map.cpp:67-120).
template <int FLAVOR>
__global__ void voxel_span_kernel(const Tables t, uint64_t i, uint64_t j, uint64_t k,
                                  uint32_t* __restrict__ be) {
  uint32_t b = 0, e = 0;
  column_span<FLAVOR>(t, i, j, k, k, &b, &e);
  be[0] = b;
  be[1] = e;
}
__global__ void voxel_ids_kernel(const PointRec* __restrict__ rec, const uint32_t* __restrict__ be,
                                 uint32_t cap, uint32_t* __restrict__ out) {
  const uint32_t b = be[0], e = be[1];
  for (uint32_t p = b + threadIdx.x; p < e && p - b < cap; p += blockDim.x) out[p - b] = rec[p].id;
}
}  // namespace apik
}  // namespace cmg

extern "C" {

// Cheesemap::voxel_present / voxel_lookup (map.hpp:62-69, map.cpp:124-136):
// *present = the voxel is materialized (always for the dense flavour; for a
// mixed map, every cell of a densified slice; otherwise non-empty); the
// voxel's handles (ascending) to `handles` (host or device, up to capacity)
// and their number to *count. Synchronous. CM_OUT_OF_DOMAIN for a voxel
// outside the grid.
cm_status cm_voxel_lookup(const cm_index* ix, uint64_t i, uint64_t j, uint64_t k, int* present,
                          uint32_t* handles, uint64_t capacity, uint64_t* count) {
  CM_TRY(check_index(ix));
  if (i >= ix->g.nx || j >= ix->g.ny || k >= ix->g.nz) {
    set_error("voxel outside the grid");
    return CM_OUT_OF_DOMAIN;
  }
  DeviceGuard dg(ix->device);
  cudaStream_t st = 0;
  uint32_t* be = nullptr;
  CM_CUDA_TRY(dev_alloc_t(&be, 2, st));
  const Tables t = ix->tables();
  if (ix->opts.flavor == CM_DENSE) apik::voxel_span_kernel<CM_DENSE><<<1, 1, 0, st>>>(t, i, j, k, be);
  else if (ix->opts.flavor == CM_SPARSE) apik::voxel_span_kernel<CM_SPARSE><<<1, 1, 0, st>>>(t, i, j, k, be);
  else apik::voxel_span_kernel<CM_MIXED><<<1, 1, 0, st>>>(t, i, j, k, be);
  ::cmg::note_launch();
  uint32_t hb[2] = {0, 0};
  CM_CUDA_TRY(cudaMemcpyAsync(hb, be, 8, cudaMemcpyDeviceToHost, st));
  CM_CUDA_TRY(cudaStreamSynchronize(st));
  const uint64_t n = hb[1] - hb[0];
  if (count) *count = n;
  if (present) {
    bool p = n > 0;
    if (ix->opts.flavor == CM_DENSE) p = true;
    if (ix->opts.flavor == CM_MIXED && k < ix->slice_ne.size())
      p = p || static_cast<double>(ix->slice_ne[k]) / static_cast<double>(ix->g.nx * ix->g.ny) >=
                   ix->opts.densify_threshold;
    *present = p ? 1 : 0;
  }
  if (handles && n && capacity) {
    OutBuf<uint32_t> h;
    CM_TRY(h.init(handles, std::min<uint64_t>(n, capacity), st));
    apik::voxel_ids_kernel<<<1, 256, 0, st>>>(ix->rec, be, (uint32_t)std::min<uint64_t>(n, capacity), h.dev);
    ::cmg::note_launch();
    CM_CUDA_TRY(cudaGetLastError());
    CM_TRY(h.finish());
  }
  dev_free(be, st);
  CM_CUDA_TRY(cudaStreamSynchronize(st));
  return CM_OK;
}

cm_status cm_corrupt_for_testing(cm_index* ix) {
  CM_TRY(check_index(ix));
  DeviceGuard dg(ix->device);
  apik::corrupt_kernel<<<1, 1, 0, 0>>>(ix->rec, ix->frec, ix->n / 2); ::cmg::note_launch();
  CM_CUDA_TRY(cudaGetLastError());
  CM_CUDA_TRY(cudaDeviceSynchronize());
  return CM_OK;
}

cm_status cm_radius_count(const cm_index* ix, const double* q, uint64_t nq, int kernel, double r,
                          uint32_t* counts, uint64_t* tested, void* stream) {
  CM_TRY(check_index(ix));
  CM_TRY(check_kernel(kernel));
  if (nq && !q) {
    set_error("null query pointer");
    return CM_INVALID_ARGUMENT;
  }
  DeviceGuard dg(ix->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  InBuf in;
  CM_TRY(stage_input(q, nq * 24, st, &in));
  OutBuf<uint32_t> c;
  OutBuf<uint64_t> t;
  CM_TRY(c.init(counts, nq, st));
  CM_TRY(t.init(tested, nq, st));
  QueryOrder ord;
  CM_TRY(order_queries(ix, static_cast<const double*>(in.dev), nq, st, &ord, r, kernel));
  CM_TRY(radius_count_dev(ix, static_cast<const double*>(in.dev), nq, kernel, r, ord.perm, c.dev,
                          t.dev, st));
  CM_TRY(c.finish());
  CM_TRY(t.finish());
  return sync_if(c.host() || t.host(), st);
}

cm_status cm_radius_fill(const cm_index* ix, const double* q, uint64_t nq, int kernel, double r,
                         const uint64_t* row_ptr, uint32_t* cols, void* stream) {
  CM_TRY(check_index(ix));
  CM_TRY(check_kernel(kernel));
  if (nq && (!q || !row_ptr)) {
    set_error("null query or row_ptr pointer");
    return CM_INVALID_ARGUMENT;
  }
  DeviceGuard dg(ix->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  InBuf in, rp;
  CM_TRY(stage_input(q, nq * 24, st, &in));
  CM_TRY(stage_input(row_ptr, (nq + 1) * 8, st, &rp));
  uint64_t nnz = 0;
  if (is_device_ptr(row_ptr)) {
    CM_CUDA_TRY(cudaMemcpyAsync(&nnz, static_cast<const uint64_t*>(rp.dev) + nq, 8,
                                cudaMemcpyDeviceToHost, st));
    CM_CUDA_TRY(cudaStreamSynchronize(st));
  } else {
    nnz = row_ptr[nq];
  }
  OutBuf<uint32_t> c;
  CM_TRY(c.init(cols, nnz, st));
  QueryOrder ord;
  CM_TRY(order_queries(ix, static_cast<const double*>(in.dev), nq, st, &ord, r, kernel));
  CM_TRY(radius_fill_dev(ix, static_cast<const double*>(in.dev), nq, kernel, r, ord.perm,
                         static_cast<const uint64_t*>(rp.dev), c.dev, st));
  CM_TRY(c.finish());
  return sync_if(c.host(), st);
}

}  // extern "C"

namespace {
struct QueryEvents {
  cudaEvent_t e[6];
  int device = 0;
  uint64_t nq = 0, nnz = 0;
  int two_pass = 0;  // 0 collect, 1 count + fill, 2 collect rerun (cm_query_timing)
  bool valid = false;
  QueryEvents() {
    cudaGetDevice(&device);
    for (auto& x : e) cudaEventCreate(&x);
  }
};
// the events of the last radius search on this thread (any device)
thread_local QueryEvents* g_last_qev = nullptr;
QueryEvents& qev() {
  QueryEvents& ev = per_thread_device<QueryEvents>();
  g_last_qev = &ev;
  return ev;
}
}  // namespace

extern "C" {

cm_status cm_get_last_query_timing(cm_query_timing* o) {
  if (!o) return CM_INVALID_ARGUMENT;
  if (!g_last_qev || !g_last_qev->valid) {
    set_error("no radius search has run on this thread");
    return CM_INVALID_ARGUMENT;
  }
  QueryEvents& ev = *g_last_qev;
  DeviceGuard dg(ev.device);
  CM_CUDA_TRY(cudaEventSynchronize(ev.e[5]));
  float ms[5], tot;
  for (int i = 0; i < 5; ++i) cudaEventElapsedTime(&ms[i], ev.e[i], ev.e[i + 1]);
  cudaEventElapsedTime(&tot, ev.e[0], ev.e[5]);
  o->order_ms = ms[0];
  o->pass1_ms = ms[1];
  o->rowsort_ms = ms[2];
  o->scan_ms = ms[3];
  o->pass2_ms = ms[4];
  o->total_ms = tot;
  o->nq = ev.nq;
  o->nnz = ev.nnz;
  o->two_pass = ev.two_pass;
  return CM_OK;
}

}  // extern "C"

namespace cmg {
namespace apik {
// A small device value -> host without the copy engines (which may be busy
// with large device->host copies queued on other streams): a one-thread
// kernel stores it into mapped pinned host memory.
__global__ void publish_u64_kernel(const unsigned long long* src, volatile unsigned long long* dst,
                                   int n) {
  for (int k = 0; k < n; ++k) dst[k] = src[k];
  __threadfence_system();
}
// dst[k] = src[idx[k]] for k < n (a few row-pointer values for the host).
__global__ void publish_gather_kernel(const uint64_t* src, const uint64_t* idx, int n,
                                      volatile unsigned long long* dst) {
  for (int k = threadIdx.x; k < n; k += blockDim.x) dst[k] = src[idx[k]];
  __threadfence_system();
}
}  // namespace apik
}  // namespace cmg

namespace {
struct MappedSlot {
  unsigned long long* host = nullptr;
  unsigned long long* dev = nullptr;
  cudaEvent_t ev = nullptr;
  bool ok = false;
  MappedSlot() {
    if (cudaHostAlloc(&host, 4096, cudaHostAllocMapped) == cudaSuccess &&
        cudaHostGetDevicePointer(reinterpret_cast<void**>(&dev), host, 0) == cudaSuccess &&
        cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) == cudaSuccess)
      ok = true;
    else
      cudaGetLastError();
  }
};
// dsrc[0..n) (n <= 2) to the host.
bool read_u64_mapped(const unsigned long long* dsrc, cudaStream_t st, unsigned long long* out,
                     int n = 1) {
  MappedSlot& slot = per_thread_device<MappedSlot>();
  if (!slot.ok) {
    if (cudaMemcpyAsync(out, dsrc, 8 * n, cudaMemcpyDeviceToHost, st) != cudaSuccess) return false;
    return cudaStreamSynchronize(st) == cudaSuccess;
  }
  cmg::apik::publish_u64_kernel<<<1, 1, 0, st>>>(dsrc, slot.dev, n); ::cmg::note_launch();
  if (cudaGetLastError() != cudaSuccess) return false;
  if (cudaEventRecord(slot.ev, st) != cudaSuccess) return false;
  if (cudaEventSynchronize(slot.ev) != cudaSuccess) return false;
  for (int k = 0; k < n; ++k) out[k] = reinterpret_cast<volatile unsigned long long*>(slot.host)[k];
  return true;
}

// row_ptr[idx[k]] for k < n (n <= 256) to the host, through mapped memory.
// idx is a host array; it travels in the mapped page too.
bool read_row_ptrs_mapped(const uint64_t* row_ptr, const uint64_t* idx, int n, cudaStream_t st,
                          uint64_t* out) {
  struct RowSlot : MappedSlot {};  // a second page per thread and device
  MappedSlot& slot = per_thread_device<RowSlot>();
  if (!slot.ok || n > 256) {
    for (int k = 0; k < n; ++k)
      if (cudaMemcpyAsync(out + k, row_ptr + idx[k], 8, cudaMemcpyDeviceToHost, st) != cudaSuccess)
        return false;
    return cudaStreamSynchronize(st) == cudaSuccess;
  }
  uint64_t* hidx = reinterpret_cast<uint64_t*>(slot.host) + 256;
  std::memcpy(hidx, idx, n * sizeof(uint64_t));
  const uint64_t* didx = reinterpret_cast<const uint64_t*>(slot.dev) + 256;
  cmg::apik::publish_gather_kernel<<<1, 256, 0, st>>>(row_ptr, didx, n, slot.dev); ::cmg::note_launch();
  if (cudaGetLastError() != cudaSuccess) return false;
  if (cudaEventRecord(slot.ev, st) != cudaSuccess) return false;
  if (cudaEventSynchronize(slot.ev) != cudaSuccess) return false;
  for (int k = 0; k < n; ++k) out[k] = reinterpret_cast<volatile unsigned long long*>(slot.host)[k];
  return true;
}

// Replaces the single gather launch of radius_search_core (to_host uses it to
// stream the CSR to the host while the gather still runs).
struct GatherHook {
  uint32_t skip_above = 0xffffffffu;  // rows longer than this were merged already
  virtual cm_status run(const uint32_t* temp, const uint64_t* toff, const uint32_t* scnt,
                        const uint64_t* row_ptr, const uint32_t* perm, uint32_t* cols, uint64_t nq,
                        cudaStream_t st) = 0;
  virtual ~GatherHook() = default;
};
}  // namespace

// count/collect + scan + gather for device-resident queries into csr's
// device buffers (row_ptr, cols, nnz). Events of the calling thread record
// the phases (cm_get_last_query_timing).
static cm_status radius_search_core(const cm_index* ix, const double* qd, uint64_t nq, int kernel,
                                    double r, cudaStream_t st, cm_csr* csr,
                                    GatherHook* hook = nullptr, const double* rq = nullptr,
                                    const double* qbox = nullptr) {
  QueryEvents& ev = qev();
  ev.valid = false;
  cudaEventRecord(ev.e[0], st);
  QueryOrder ord;
  CM_TRY(order_queries(ix, qd, nq, st, &ord, r, kernel));
  qd = ord.q;  // null for self queries read from the records
  cudaEventRecord(ev.e[1], st);
  uint32_t* counts = nullptr;
  uint64_t* toff = nullptr;
  uint32_t* scnt = nullptr;
  uint32_t* temp = nullptr;
  unsigned long long* cursor = nullptr;
  auto release = [&]() {
    if (counts) dev_free(counts, st);
    if (toff) dev_free(toff, st);
    if (scnt) dev_free(scnt, st);
    if (temp) dev_free(temp, st);
    if (cursor) dev_free(cursor, st);
    counts = nullptr, toff = nullptr, scnt = nullptr, temp = nullptr, cursor = nullptr;
  };
  auto fail = [&](cm_status s) {
    release();
    cudaStreamSynchronize(st);
    return s;
  };
  MergeList ml;
  ml.st = st;
  if (dev_alloc_t(&counts, nq + 1, st) != cudaSuccess ||
      dev_alloc_t(&ml.off, nq + 1, st) != cudaSuccess ||
      dev_alloc_t(&ml.len, nq + 1, st) != cudaSuccess ||
      dev_alloc_t(&ml.q, nq + 1, st) != cudaSuccess || dev_alloc_t(&ml.n, 1, st) != cudaSuccess ||
      dev_alloc_t(&csr->row_ptr, nq + 1, st) != cudaSuccess ||
      dev_alloc_t(&toff, nq + 1, st) != cudaSuccess || dev_alloc_t(&scnt, nq + 1, st) != cudaSuccess ||
      dev_alloc_t(&cursor, 2, st) != cudaSuccess) {
    set_error("device allocation failed (row pointers)");
    return fail(CM_CUDA);
  }
  // Single pass: sorted rows into an arena sized from the running
  // neighbours-per-query estimate; if the arena overflows, fall back to
  // count + scan + fill.
  // Large radii go count + scan + fill (wide tiles) + in-place row sort.
  // An overflowing collect still counts every reservation, so the cursor
  // then holds the exact arena size: the collect reruns once into an arena of
  // that size (query subsets differ in density, e.g. the chunks of a
  // host-buffer call over a cloud generated ground first, buildings last).
  const double est = ix->nnz_per_query.load(std::memory_order_relaxed);
  uint64_t cap = (uint64_t)((double)nq * est * 1.25) + (1u << 20);
  bool two_pass = radius_is_wide(ix, r);
  if (!two_pass && dev_alloc_t(&temp, cap, st) != cudaSuccess) {
    two_pass = true;
    cudaGetLastError();
  }
  cm_status s = CM_OK;
  unsigned long long used = 0;        // arena entries (rows padded to 4 handles)
  unsigned long long cur[2] = {0, 0}; // arena cursor, exact handle count
  bool recollected = false;
  if (!two_pass) {
    s = radius_collect_dev(ix, qd, nq, kernel, r, ord.perm, temp, cap, toff, scnt, counts, cursor,
                           st, ev.e[2], rq, qbox, &ml);
    cudaEventRecord(ev.e[3], st);
    if (s != CM_OK) return fail(s);
    if (!read_u64_mapped(cursor, st, cur, 2)) {
      set_error("arena cursor readback failed");
      return fail(CM_CUDA);
    }
    used = cur[0];
    // slow decay: alternating dense and sparse batches keep the larger size
    if (nq)
      ix->nnz_per_query.store(std::max({1.0, (double)used / (double)nq, 0.95 * est}),
                              std::memory_order_relaxed);
    if (used > cap && !std::getenv("CMGPU_NO_RECOLLECT")) {
      dev_free(temp, st);
      temp = nullptr;
      cap = used;
      if (dev_alloc_t(&temp, cap, st) == cudaSuccess) {
        recollected = true;
        s = radius_collect_dev(ix, qd, nq, kernel, r, ord.perm, temp, cap, toff, scnt, counts,
                               cursor, st, ev.e[2], rq, qbox, &ml);
        cudaEventRecord(ev.e[3], st);
        if (s != CM_OK) return fail(s);
        if (!read_u64_mapped(cursor, st, cur, 2)) {
          set_error("arena cursor readback failed");
          return fail(CM_CUDA);
        }
        used = cur[0];
      } else {
        cudaGetLastError();
      }
    }
    two_pass = used > cap || !temp;
    if (two_pass && temp) {
      dev_free(temp, st);
      temp = nullptr;
    }
  }
  if (two_pass) {
    cudaEventRecord(ev.e[1], st);
    s = radius_count_dev(ix, qd, nq, kernel, r, ord.perm, counts, nullptr, st, rq, qbox);
    cudaEventRecord(ev.e[2], st);
    cudaEventRecord(ev.e[3], st);
    if (s != CM_OK) return fail(s);
  }
  s = counts_to_row_ptr(counts, nq, csr->row_ptr, st);
  cudaEventRecord(ev.e[4], st);
  if (s != CM_OK) return fail(s);
  // Row-sort plan of a wide FILL: rows of 513..1024 go to the merge-path
  // block sort when they are short on average (config 1 cube r = 2.5, class
  // mean 624: fill + sort 158 -> 142 ms), else to the 512-head split sort,
  // which measured faster for longer class means (sphere / cube r = 5, 703 /
  // 930: 37.7 / 50.0 -> 36.7 / 46.0 ms on 2M centres; sphere r = 2.5, 692:
  // equal). The threshold sits between the measured cases.
  uint32_t mid_min = 0;
  if (two_pass) {
    unsigned long long cls_h[2] = {0, 0};
    unsigned long long* cls_d = nullptr;
    const bool cls = dev_alloc_t(&cls_d, 2, st) == cudaSuccess &&
                     row_class_counts_dev(counts, nq, cls_d, st) == CM_OK &&
                     cudaMemcpyAsync(cls_h, cls_d, 16, cudaMemcpyDeviceToHost, st) == cudaSuccess;
    if (cudaMemcpyAsync(&csr->nnz, csr->row_ptr + nq, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess) {
      set_error("row pointer readback failed");
      if (cls_d) dev_free(cls_d, st);
      return fail(CM_CUDA);
    }
    if (cls_d) dev_free(cls_d, st);
    cudaGetLastError();
    if (cls && cls_h[0] > 0 && (double)cls_h[1] / (double)cls_h[0] < 660.0) mid_min = 512;
  } else {
    csr->nnz = cur[1];
  }
  if (dev_alloc_t(&csr->cols, csr->nnz, st) != cudaSuccess) {
    set_error("device allocation failed (columns)");
    return fail(CM_CUDA);
  }
  if (two_pass)
    s = radius_fill_dev(ix, qd, nq, kernel, r, ord.perm, csr->row_ptr, csr->cols, st, nullptr,
                        mid_min, rq, qbox);
  else {
    // long rows: merged from their sorted voxel runs straight into the CSR
    // (before the gather, so a streaming hook copies finished rows)
    s = merge_big_rows(ml, temp, csr->row_ptr, csr->cols, st);
    if (s == CM_OK) {
      if (hook) {
        hook->skip_above = long_row_min() - 1;
        s = hook->run(temp, toff, scnt, csr->row_ptr, ord.perm, csr->cols, nq, st);
      } else {
        s = gather_rows_dev(temp, toff, scnt, csr->row_ptr, ord.perm, csr->cols, nq, st,
                            long_row_min() - 1);
      }
    }
  }
  cudaEventRecord(ev.e[5], st);
  if (s != CM_OK) return fail(s);
  ev.nq = nq;
  ev.nnz = csr->nnz;
  ev.two_pass = two_pass ? 1 : recollected ? 2 : 0;
  ev.valid = true;
  release();
  return CM_OK;
}


extern "C" {

cm_status cm_radius_search(const cm_index* ix, const double* q, uint64_t nq, int kernel, double r,
                           void* stream, cm_csr** out) {
  CM_TRY(check_index(ix));
  CM_TRY(check_kernel(kernel));
  if (!out || (nq && !q)) {
    set_error("null query or output pointer");
    return CM_INVALID_ARGUMENT;
  }
  *out = nullptr;
  DeviceGuard dg(ix->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  InBuf in;
  CM_TRY(stage_input(q, nq * 24, st, &in));
  cm_csr* csr = new cm_csr();
  csr->nq = nq;
  csr->device = ix->device;
  const cm_status s = radius_search_core(ix, static_cast<const double*>(in.dev), nq, kernel, r,
                                         st, csr);
  if (s != CM_OK) {
    cm_csr_free(csr);
    return s;
  }
  *out = csr;
  return CM_OK;
}

// Every indexed point as a centre (the "every point is a query" workloads of
// SURVEY.md §8d configs 1 and 4): row q is the result for point q. The
// centres are read from the index's own cell-ordered records, so no query
// sort runs and the caller passes no buffer.
cm_status cm_radius_search_self(const cm_index* ix, int kernel, double r, void* stream,
                                cm_csr** out) {
  CM_TRY(check_index(ix));
  CM_TRY(check_kernel(kernel));
  if (!out) {
    set_error("null output pointer");
    return CM_INVALID_ARGUMENT;
  }
  *out = nullptr;
  if (ix->global_ids) {
    set_error("self queries of a slab index: use cm_slab_radius_search (owned centres)");
    return CM_INVALID_ARGUMENT;
  }
  DeviceGuard dg(ix->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cm_csr* csr = new cm_csr();
  csr->nq = ix->n;
  csr->device = ix->device;
  const cm_status s = radius_search_core(ix, nullptr, ix->n, kernel, r, st, csr);
  if (s != CM_OK) {
    cm_csr_free(csr);
    return s;
  }
  *out = csr;
  return CM_OK;
}

}  // extern "C"

namespace cmg {
namespace apik {
// Explicit kernels -> centres (query order only), per-centre radius, and
// the kernel's box() where it is not c +- r:
//   CM_SPHERE   4 doubles: cx cy cz r            (box c +- r, computed by the kernels)
//   CM_CUBE     6 doubles: min xyz, max xyz      (BoxKernel{Aabb}, geometry.hpp:87-92)
//   CM_CYLINDER 5 doubles: cx cy r z_lo z_hi     (geometry.hpp:97-113)
__global__ void kernel_params_kernel(int kind, const double* __restrict__ prm, uint64_t nq,
                                     DevGrid g, double* __restrict__ q, double* __restrict__ rq,
                                     double* __restrict__ qbox) {
  const int w = kind == CM_SPHERE ? 4 : kind == CM_CUBE ? 6 : 5;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nq;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const double* p = prm + (uint64_t)w * i;
    double cx, cy, cz, r = 0.0;
    if (kind == CM_SPHERE) {
      cx = p[0], cy = p[1], cz = p[2], r = p[3];
    } else if (kind == CM_CUBE) {
      double* b = qbox + 6 * i;
      for (int a = 0; a < 6; ++a) b[a] = p[a];
      cx = 0.5 * (p[0] + p[3]), cy = 0.5 * (p[1] + p[4]), cz = 0.5 * (p[2] + p[5]);
    } else {
      cx = p[0], cy = p[1], r = p[2];
      double* b = qbox + 6 * i;
      b[0] = __dsub_rn(cx, r), b[1] = __dsub_rn(cy, r), b[2] = p[3];
      b[3] = __dadd_rn(cx, r), b[4] = __dadd_rn(cy, r), b[5] = p[4];
      cz = 0.5 * (fmax(p[3], g.bz0) + fmin(p[4], g.bz1));
    }
    // A box's centre only orders the queries (its predicate reads the box),
    // so it is kept finite and inside the grid; sphere centres and the
    // cylinder's axis are the predicates' own and pass unchanged.
    if (kind == CM_CUBE) {
      cx = fmin(fmax(cx, g.bx0), g.bx1);
      cy = fmin(fmax(cy, g.by0), g.by1);
      cx = isnan(cx) ? g.bx0 : cx;
      cy = isnan(cy) ? g.by0 : cy;
    }
    if (kind != CM_SPHERE) {
      cz = fmin(fmax(cz, g.bz0), g.bz1);
      cz = isnan(cz) ? g.bz0 : cz;
    }
    q[3 * i] = cx;
    q[3 * i + 1] = cy;
    q[3 * i + 2] = cz;
    rq[i] = r;
  }
}

// QueryStats::voxels_visited (search.hpp:116-119): the voxels of the
// kernel's clamped range, empty or not.
__global__ void voxels_visited_kernel(int kind, const double* __restrict__ q,
                                      const double* __restrict__ rq, const double* __restrict__ qbox,
                                      uint64_t nq, DevGrid g, uint64_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nq;
       i += (uint64_t)gridDim.x * blockDim.x) {
    Range R;
    const bool ok = clamped_range(g, q[3 * i], q[3 * i + 1], q[3 * i + 2], rq[i], &R, kind,
                                  kind == CM_SPHERE ? nullptr : qbox + 6 * i);
    out[i] = ok ? (R.i1 - R.i0 + 1) * (R.j1 - R.j0 + 1) * (R.k1 - R.k0 + 1) : 0;
  }
}
}  // namespace apik
}  // namespace cmg

namespace {
// Device buffers of an explicit-kernel batch (kernel_params_kernel).
struct KernelBatch {
  double* q = nullptr;
  double* rq = nullptr;
  double* qbox = nullptr;
  cudaStream_t st = nullptr;
  ~KernelBatch() {
    if (q) dev_free(q, st);
    if (rq) dev_free(rq, st);
    if (qbox) dev_free(qbox, st);
  }
  cm_status init(const cm_index* ix, int kind, const double* params, uint64_t nq, cudaStream_t s) {
    st = s;
    if (kind != CM_SPHERE && kind != CM_CUBE && kind != CM_CYLINDER) {
      set_error("unknown kernel (CM_SPHERE = 0, CM_CUBE = 1 (Aabb box), CM_CYLINDER = 2)");
      return CM_INVALID_ARGUMENT;
    }
    const int w = kind == CM_SPHERE ? 4 : kind == CM_CUBE ? 6 : 5;
    InBuf in;
    CM_TRY(stage_input(params, nq * w * 8, st, &in));
    CM_CUDA_TRY(dev_alloc_t(&q, 3 * nq + 3, st));
    CM_CUDA_TRY(dev_alloc_t(&rq, nq + 1, st));
    if (kind != CM_SPHERE) CM_CUDA_TRY(dev_alloc_t(&qbox, 6 * nq + 6, st));
    if (nq) {
      const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((nq + 255) / 256, (uint64_t)sm_count() * 8));
      apik::kernel_params_kernel<<<grid, 256, 0, st>>>(kind, static_cast<const double*>(in.dev), nq,
                                                       ix->g, q, rq, qbox);
      ::cmg::note_launch();
      CM_CUDA_TRY(cudaGetLastError());
    }
    return CM_OK;
  }
};
}  // namespace

extern "C" {

// kernel_search (search.hpp:102-127) for a batch of explicit kernels, each
// with its own parameters (see kernel_params_kernel): per-centre radii,
// BoxKernel Aabbs, bounded cylinders. Sorted rows like cm_radius_search.
cm_status cm_kernel_search(const cm_index* ix, int kernel, const double* params, uint64_t nq,
                           void* stream, cm_csr** out) {
  CM_TRY(check_index(ix));
  if (!out || (nq && !params)) {
    set_error("null parameters or output pointer");
    return CM_INVALID_ARGUMENT;
  }
  *out = nullptr;
  DeviceGuard dg(ix->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  KernelBatch kb;
  CM_TRY(kb.init(ix, kernel, params, nq, st));
  cm_csr* csr = new cm_csr();
  csr->nq = nq;
  csr->device = ix->device;
  const cm_status s =
      radius_search_core(ix, kb.q, nq, kernel, -1.0, st, csr, nullptr, kb.rq, kb.qbox);
  if (s != CM_OK) {
    cm_csr_free(csr);
    return s;
  }
  *out = csr;
  return CM_OK;
}

// Counts and QueryStats (search.hpp:12-17) of explicit kernels: counts[q],
// points_tested[q], voxels_visited[q]; any output may be NULL; host or
// device outputs.
cm_status cm_kernel_count(const cm_index* ix, int kernel, const double* params, uint64_t nq,
                          uint32_t* counts, uint64_t* points_tested, uint64_t* voxels_visited,
                          void* stream) {
  CM_TRY(check_index(ix));
  if (nq && !params) {
    set_error("null parameters");
    return CM_INVALID_ARGUMENT;
  }
  DeviceGuard dg(ix->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  KernelBatch kb;
  CM_TRY(kb.init(ix, kernel, params, nq, st));
  OutBuf<uint32_t> c;
  OutBuf<uint64_t> t, v;
  CM_TRY(c.init(counts, nq, st));
  CM_TRY(t.init(points_tested, nq, st));
  CM_TRY(v.init(voxels_visited, nq, st));
  if (nq && (c.dev || t.dev)) {
    QueryOrder ord;
    CM_TRY(order_queries(ix, kb.q, nq, st, &ord, -1.0, kernel));
    CM_TRY(radius_count_dev(ix, kb.q, nq, kernel, -1.0, ord.perm, c.dev, t.dev, st, kb.rq,
                            kb.qbox));
  }
  if (nq && v.dev) {
    const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((nq + 255) / 256, (uint64_t)sm_count() * 8));
    apik::voxels_visited_kernel<<<grid, 256, 0, st>>>(kernel, kb.q, kb.rq, kb.qbox, nq, ix->g, v.dev);
    ::cmg::note_launch();
    CM_CUDA_TRY(cudaGetLastError());
  }
  CM_TRY(c.finish());
  CM_TRY(t.finish());
  CM_TRY(v.finish());
  return sync_if(c.host() || t.host() || v.host(), st);
}

namespace {
// One-chunk to_host: once the row pointers are scanned, the gather runs in G
// query ranges and each range's columns start their device->host copy as
// soon as that range is gathered (the row pointers go first), so the PCIe
// copy of the CSR overlaps the gather.
struct StreamingGather : GatherHook {
  static constexpr int G = 8;
  cudaStream_t out = nullptr;
  uint64_t* row_ptr_host = nullptr;
  uint32_t* cols_host = nullptr;
  uint64_t cap = 0;        // columns the host buffer still holds
  bool rows_early = true;  // copy the row pointers before the columns (chunk 0 only:
                           // later chunks' rows need the running offset first)
  bool copied = false, over = false;
  uint64_t nnz = 0;
  cm_status run(const uint32_t* temp, const uint64_t* toff, const uint32_t* scnt,
                const uint64_t* row_ptr, const uint32_t* perm, uint32_t* cols, uint64_t nq,
                cudaStream_t st) override {
    struct Events {
      cudaEvent_t e[G + 1];
      Events() {
        for (auto& x : e) cudaEventCreateWithFlags(&x, cudaEventDisableTiming);
      }
    };
    Events& evs = per_thread_device<Events>();
    uint64_t qb[G + 1], rp[G + 1];
    for (int k = 0; k <= G; ++k) qb[k] = nq * (uint64_t)k / G;
    if (!read_row_ptrs_mapped(row_ptr, qb, G + 1, st, rp)) {
      set_error("row pointer readback failed");
      return CM_CUDA;
    }
    nnz = rp[G];
    over = nnz > cap;
    if (rows_early) {
      CM_CUDA_TRY(cudaEventRecord(evs.e[G], st));
      CM_CUDA_TRY(cudaStreamWaitEvent(out, evs.e[G], 0));
      CM_CUDA_TRY(cudaMemcpyAsync(row_ptr_host + 1, row_ptr + 1, nq * 8, cudaMemcpyDeviceToHost, out));
    }
    for (int k = 0; k < G; ++k) {
      if (qb[k + 1] == qb[k]) continue;
      CM_TRY(gather_rows_dev(temp, toff + qb[k], scnt + qb[k], row_ptr + qb[k], perm, cols,
                             qb[k + 1] - qb[k], st, skip_above));
      if (!over && rp[k + 1] > rp[k]) {
        CM_CUDA_TRY(cudaEventRecord(evs.e[k], st));
        CM_CUDA_TRY(cudaStreamWaitEvent(out, evs.e[k], 0));
        CM_CUDA_TRY(cudaMemcpyAsync(cols_host + rp[k], cols + rp[k], (rp[k + 1] - rp[k]) * 4,
                                    cudaMemcpyDeviceToHost, out));
      }
    }
    copied = true;
    return CM_OK;
  }
};
}  // namespace

// Host-buffer pipeline: queries in chunks (three streams): all input copies
// are issued up front, and chunk i's CSR copy to the host overlaps its own
// gather and chunk i+1's kernels. row_ptr_host gets nq + 1 entries, cols_host up to cols_capacity.
cm_status cm_radius_search_to_host(const cm_index* ix, const double* q_host, uint64_t nq,
                                   int kernel, double r, uint64_t* row_ptr_host,
                                   uint32_t* cols_host, uint64_t cols_capacity, uint64_t* nnz_out,
                                   void* stream) {
  CM_TRY(check_index(ix));
  CM_TRY(check_kernel(kernel));
  if ((nq && !q_host) || !row_ptr_host || !nnz_out) {
    set_error("null query or output pointer");
    return CM_INVALID_ARGUMENT;
  }
  DeviceGuard dg(ix->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  struct Streams {
    cudaStream_t in = nullptr, out = nullptr;
    Streams() {  // per host thread, kept for the process lifetime
      cudaStreamCreateWithFlags(&in, cudaStreamNonBlocking);
      cudaStreamCreateWithFlags(&out, cudaStreamNonBlocking);
    }
  };
  Streams& ss = per_thread_device<Streams>();
  // Every chunk's CSR streams to the host while its gather runs, and chunk
  // i+1's input copy and kernels overlap chunk i's columns on PCIe, which
  // bounds the call (~54 GB/s device->host vs ~1 G queries/s of kernels).
  // Query tiles form within a chunk, so a chunk is a sparser sample of the
  // batch (config 1: 5M-query chunks run ~25 % slower per query, hidden
  // behind the copy). 4 chunks of >= 4M queries measured best (config 1:
  // 88 -> 74 ms per call); CMGPU_CHUNKS overrides.
  uint64_t nchunks = std::min<uint64_t>(4, std::max<uint64_t>(1, nq / (4u << 20)));
  if (const char* ev = std::getenv("CMGPU_CHUNKS")) nchunks = std::max<uint64_t>(1, std::strtoull(ev, nullptr, 10));
  // Chunk boundaries: the first chunk is a third of the size of the others,
  // so the first columns reach PCIe sooner (config 1, weights 1:2:2:2 / 1:3:3:3
  // / 1:2:4:4:4: 67.55 / 66.97 / 67.1 ms per call).
  std::vector<uint64_t> qb(nchunks + 1);
  std::vector<double> w(nchunks, 3.0);
  w[0] = 1.0;
  if (const char* rv = std::getenv("CMGPU_CHUNK_W")) {  // e.g. "1,2,4,4,4" (probe)
    w.clear();
    for (const char* p = rv; *p;) {
      char* e = nullptr;
      w.push_back(std::strtod(p, &e));
      p = *e ? e + 1 : e;
    }
    nchunks = w.size();
    qb.assign(nchunks + 1, 0);
  }
  double wsum = 0.0;
  for (double x : w) wsum += x;
  double acc = 0.0;
  for (uint64_t c = 0; c < nchunks; ++c) {
    qb[c] = (uint64_t)((double)nq * acc / wsum);
    acc += w[c];
  }
  qb[nchunks] = nq;
  double* qdev = nullptr;  // every chunk's input copy is issued up front
  std::vector<cudaEvent_t> in_done(nchunks);  // sized after the chunk plan
  cudaEvent_t comp_done[2], out_done[2];
  // CMGPU_TRACE: device timeline per chunk (core start / core end on the
  // compute stream, copies done on the output stream), relative to t_ev[0]
  constexpr int kTraceChunks = 16;
  cudaEvent_t t_ev[1 + 3 * kTraceChunks] = {};
  for (auto& e : in_done) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  for (int i = 0; i < 2; ++i) {
    cudaEventCreateWithFlags(&comp_done[i], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&out_done[i], cudaEventDisableTiming);
  }
  cm_csr csrs[2];
  cm_status s = CM_OK;
  if (nq && dev_alloc_t(&qdev, nq * 3, ss.in) != cudaSuccess) s = CM_CUDA;
  uint64_t base = 0;
  bool full = false;
  row_ptr_host[0] = 0;
  static const bool trace = std::getenv("CMGPU_TRACE") != nullptr;
  if (trace) {
    for (auto& e : t_ev) cudaEventCreate(&e);
    cudaEventRecord(t_ev[0], st);
  }
  auto mark = [&](uint64_t c, int what, cudaStream_t on) {
    if (trace && c < (uint64_t)kTraceChunks) cudaEventRecord(t_ev[1 + 3 * c + what], on);
  };
  if (trace) cudaStreamWaitEvent(ss.in, t_ev[0], 0);
  for (uint64_t c = 0; s == CM_OK && c < nchunks; ++c) {
    cudaMemcpyAsync(qdev + 3 * qb[c], q_host + 3 * qb[c], (qb[c + 1] - qb[c]) * 24,
                    cudaMemcpyHostToDevice, ss.in);
    cudaEventRecord(in_done[c], ss.in);
    mark(c, 0, ss.in);
  }
  auto t0 = std::chrono::steady_clock::now();
  auto tr = [&](const char* what, uint64_t c) {
    if (trace)
      std::fprintf(stderr, "[to_host] %8.3f ms chunk %lu %s\n",
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(),
                   (unsigned long)c, what);
  };
  for (uint64_t c = 0; s == CM_OK && c < nchunks; ++c) {
    const uint64_t q0 = qb[c], n = qb[c + 1] - qb[c];
    const int bi = (int)(c & 1);
    if (n == 0) continue;
    tr("start", c);
    cudaStreamWaitEvent(st, in_done[c], 0);
    cudaStreamWaitEvent(st, out_done[bi], 0);  // csrs[bi] no longer being copied
    if (csrs[bi].row_ptr) {
      dev_free(csrs[bi].row_ptr, st);
      dev_free(csrs[bi].cols, st);
      csrs[bi].row_ptr = nullptr, csrs[bi].cols = nullptr;
    }
    csrs[bi].nq = n;
    csrs[bi].device = ix->device;
    StreamingGather sg;
    sg.out = ss.out;
    sg.row_ptr_host = row_ptr_host + q0;
    sg.cols_host = cols_host + (full ? 0 : base);
    sg.cap = full || base > cols_capacity ? 0 : cols_capacity - base;
    sg.rows_early = base == 0;
    s = radius_search_core(ix, qdev + 3 * q0, n, kernel, r, st, &csrs[bi], &sg);
    tr("core returned", c);
    mark(c, 1, st);
    if (trace) {
      cm_query_timing qt;
      cm_get_last_query_timing(&qt);
      std::fprintf(stderr, "   device: order %.2f pass1 %.2f scan %.2f pass2 %.2f total %.2f ms\n",
                   qt.order_ms, qt.pass1_ms, qt.scan_ms, qt.pass2_ms, qt.total_ms);
    }
    if (s != CM_OK) break;
    if (base) {
      apik::add_offset_kernel<<<(unsigned)std::min<uint64_t>((n + 255) / 256, 4096), 256, 0, st>>>(
          csrs[bi].row_ptr + 1, n, base); ::cmg::note_launch();
    }
    cudaEventRecord(comp_done[bi], st);
    if (sg.copied) {  // columns streamed during the gather
      full = full || sg.over;
      if (!sg.rows_early) {
        cudaStreamWaitEvent(ss.out, comp_done[bi], 0);
        cudaMemcpyAsync(row_ptr_host + q0 + 1, csrs[bi].row_ptr + 1, n * 8, cudaMemcpyDeviceToHost,
                        ss.out);
      }
      cudaEventRecord(out_done[bi], ss.out);
      mark(c, 2, ss.out);
      base += csrs[bi].nnz;
      continue;
    }
    full = full || base + csrs[bi].nnz > cols_capacity;  // keep counting: report the size needed
    // rows of this chunk (already offset by `base` on the device)
    cudaStreamWaitEvent(ss.out, comp_done[bi], 0);
    cudaMemcpyAsync(row_ptr_host + q0 + 1, csrs[bi].row_ptr + 1, n * 8, cudaMemcpyDeviceToHost,
                    ss.out);
    if (csrs[bi].nnz && !full)
      cudaMemcpyAsync(cols_host + base, csrs[bi].cols, csrs[bi].nnz * 4, cudaMemcpyDeviceToHost,
                      ss.out);
    cudaEventRecord(out_done[bi], ss.out);
    base += csrs[bi].nnz;
  }
  cudaStreamSynchronize(ss.out);
  cudaStreamSynchronize(st);
  tr("all done", 0);
  if (trace) {
    for (uint64_t c = 0; c < std::min<uint64_t>(nchunks, kTraceChunks); ++c) {
      float a = -1, b = -1, d = -1;
      cudaEventElapsedTime(&a, t_ev[0], t_ev[1 + 3 * c]);
      cudaEventElapsedTime(&b, t_ev[0], t_ev[1 + 3 * c + 1]);
      cudaEventElapsedTime(&d, t_ev[0], t_ev[1 + 3 * c + 2]);
      std::fprintf(stderr, "[to_host dev] chunk %lu: input copied %.2f  core done %.2f  copies done %.2f ms\n",
                   (unsigned long)c, a, b, d);
    }
    cudaGetLastError();
    for (auto& e : t_ev) cudaEventDestroy(e);
  }
  *nnz_out = base;
  if (s == CM_OK && full) s = CM_CAPACITY;
  if (s == CM_CAPACITY) {
    set_error("cols_capacity too small; *nnz_out holds the size needed");
  }
  for (auto& e : in_done) {
    cudaStreamWaitEvent(st, e, 0);  // an early exit may leave input copies in flight
    cudaEventDestroy(e);
  }
  if (qdev) dev_free(qdev, st);
  for (int i = 0; i < 2; ++i) {
    if (csrs[i].row_ptr) dev_free(csrs[i].row_ptr, st);
    if (csrs[i].cols) dev_free(csrs[i].cols, st);
    cudaEventDestroy(comp_done[i]);
    cudaEventDestroy(out_done[i]);
  }
  cudaStreamSynchronize(st);
  return s;
}

cm_status cm_csr_info(const cm_csr* csr, uint64_t* nq, uint64_t* nnz, const uint64_t** row_ptr,
                      const uint32_t** cols) {
  if (!csr) {
    set_error("null csr");
    return CM_INVALID_ARGUMENT;
  }
  if (nq) *nq = csr->nq;
  if (nnz) *nnz = csr->nnz;
  if (row_ptr) *row_ptr = csr->row_ptr;
  if (cols) *cols = csr->cols;
  return CM_OK;
}

cm_status cm_csr_download(const cm_csr* csr, uint64_t* row_ptr, uint32_t* cols, void* stream) {
  if (!csr) {
    set_error("null csr");
    return CM_INVALID_ARGUMENT;
  }
  DeviceGuard dg(csr->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (row_ptr)
    CM_CUDA_TRY(cudaMemcpyAsync(row_ptr, csr->row_ptr, (csr->nq + 1) * 8, cudaMemcpyDefault, st));
  if (cols && csr->nnz)
    CM_CUDA_TRY(cudaMemcpyAsync(cols, csr->cols, csr->nnz * 4, cudaMemcpyDefault, st));
  CM_CUDA_TRY(cudaStreamSynchronize(st));
  return CM_OK;
}

cm_status cm_csr_free(cm_csr* csr) {
  if (!csr) return CM_OK;
  DeviceGuard dg(csr->device);
  cudaDeviceSynchronize();
  if (csr->row_ptr) cudaFreeAsync(csr->row_ptr, 0);
  if (csr->cols) cudaFreeAsync(csr->cols, 0);
  cudaStreamSynchronize(0);
  delete csr;
  return CM_OK;
}

cm_status cm_radius_digest(const cm_index* ix, const double* q, uint64_t nq, int kernel, double r,
                           uint32_t* counts, uint64_t* digests, void* stream) {
  CM_TRY(check_index(ix));
  CM_TRY(check_kernel(kernel));
  if (nq && (!q || !counts || !digests)) {
    set_error("null query or output pointer");
    return CM_INVALID_ARGUMENT;
  }
  DeviceGuard dg(ix->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  InBuf in;
  CM_TRY(stage_input(q, nq * 24, st, &in));
  OutBuf<uint32_t> c;
  OutBuf<uint64_t> d;
  CM_TRY(c.init(counts, nq, st));
  CM_TRY(d.init(digests, nq, st));
  QueryOrder ord;
  CM_TRY(order_queries(ix, static_cast<const double*>(in.dev), nq, st, &ord, r, kernel));
  CM_TRY(radius_digest_dev(ix, static_cast<const double*>(in.dev), nq, kernel, r, ord.perm, c.dev,
                           d.dev, st));
  CM_TRY(c.finish());
  CM_TRY(d.finish());
  return sync_if(c.host() || d.host(), st);
}

// Verification of a device CSR (row_ptr, cols in device memory): per-row
// count and digest as cm_radius_digest reports them, and the number of rows
// that are not strictly ascending (to *unsorted_rows, host memory).
cm_status cm_csr_digest(const uint64_t* row_ptr, const uint32_t* cols, uint64_t nq,
                        uint32_t* counts, uint64_t* digests, uint64_t* unsorted_rows,
                        void* stream) {
  if (!row_ptr || (nq && !cols) || !unsorted_rows) {
    set_error("null CSR or output pointer");
    return CM_INVALID_ARGUMENT;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  unsigned long long* dbad = nullptr;
  CM_CUDA_TRY(dev_alloc_t(&dbad, 1, st));
  cm_status s = csr_digest_dev(row_ptr, cols, nq, counts, digests, dbad, st);
  unsigned long long h = 0;
  if (s == CM_OK && cudaMemcpyAsync(&h, dbad, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess)
    s = CM_CUDA;
  cudaFreeAsync(dbad, st);
  if (s == CM_OK && cudaStreamSynchronize(st) != cudaSuccess) s = CM_CUDA;
  *unsorted_rows = h;
  return s;
}

// brute_radius (baseline.hpp:11-21) on the device: (count, digest) per centre.
cm_status cm_brute_radius(const double* xyz, uint64_t n, const double* q, uint64_t nq, int kernel,
                          double r, uint32_t* counts, uint64_t* digests, int device, void* stream) {
  CM_TRY(check_kernel(kernel));
  if ((n && !xyz) || (nq && (!q || !counts || !digests))) {
    set_error("null point, query or output pointer");
    return CM_INVALID_ARGUMENT;
  }
  DeviceGuard dg(device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  InBuf pin, qin;
  CM_TRY(stage_input(xyz, n * 24, st, &pin));
  CM_TRY(stage_input(q, nq * 24, st, &qin));
  OutBuf<uint32_t> c;
  OutBuf<uint64_t> d;
  CM_TRY(c.init(counts, nq, st));
  CM_TRY(d.init(digests, nq, st));
  CM_TRY(brute_radius_dev(static_cast<const double*>(pin.dev), n, static_cast<const double*>(qin.dev),
                          nq, kernel, r, c.dev, d.dev, st));
  CM_TRY(c.finish());
  CM_TRY(d.finish());
  return sync_if(c.host() || d.host(), st);
}

// brute_knn (baseline.cpp:8-25) on the device, ordered by (d², handle);
// k <= 64. Missing neighbours (k > n) are handle 0xffffffff, d² = +inf.
cm_status cm_brute_knn(const double* xyz, uint64_t n, const double* q, uint64_t nq, uint32_t k,
                       uint32_t* idx, double* d2, int device, void* stream) {
  if (k == 0) {
    set_error("k must be at least 1");
    return CM_INVALID_ARGUMENT;
  }
  if (k > (uint32_t)kBruteKMax) {
    set_error("brute-force kNN supports k <= 64");
    return CM_INVALID_ARGUMENT;
  }
  if ((n && !xyz) || (nq && (!q || !idx || !d2))) {
    set_error("null point, query or output pointer");
    return CM_INVALID_ARGUMENT;
  }
  DeviceGuard dg(device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  InBuf pin, qin;
  CM_TRY(stage_input(xyz, n * 24, st, &pin));
  CM_TRY(stage_input(q, nq * 24, st, &qin));
  OutBuf<uint32_t> oi;
  OutBuf<double> od;
  CM_TRY(oi.init(idx, nq * k, st));
  CM_TRY(od.init(d2, nq * k, st));
  CM_TRY(brute_knn_dev(static_cast<const double*>(pin.dev), n, static_cast<const double*>(qin.dev),
                       nq, k, oi.dev, od.dev, st));
  CM_TRY(oi.finish());
  CM_TRY(od.finish());
  return sync_if(oi.host() || od.host(), st);
}

// global_density (analysis.cpp:17-24): points per m^2 of the xy bounding
// rectangle, from a device-built index's bounds.
cm_status cm_global_density(const double* xyz, uint64_t n, int device, void* stream,
                            double* value) {
  if (!value) {
    set_error("null output");
    return CM_INVALID_ARGUMENT;
  }
  cm_build_options o;
  cm_default_options(&o);
  o.flavor = CM_SPARSE;
  o.mode = CM_TWOD;
  cm_index* ix = nullptr;
  CM_TRY(cm_build(xyz, n, &o, device, stream, &ix));
  const DevGrid& g = ix->g;
  const double area = (g.bx1 - g.bx0) * (g.by1 - g.by0);
  cm_free(ix);
  if (!(area > 0.0)) {
    set_error("bounding rectangle has zero area");
    return CM_INVALID_ARGUMENT;
  }
  *value = static_cast<double>(n) / area;
  return CM_OK;
}

// weighted_density (analysis.cpp:26-86) on the device: the seeded subsample
// (host, the reference's partial Fisher-Yates over mt19937_64), a 2D sparse
// map at 1 m, cylinder counts for every sampled point (the COUNT pass with
// CM_CYLINDER r = 1), then the 256-bin histogram and its weighted mean.
cm_status cm_weighted_density(const double* xyz, uint64_t n, uint64_t sample_size, uint64_t seed,
                              int device, void* stream, double* value, uint64_t* bins256) {
  if (!value || !bins256) {
    set_error("null output");
    return CM_INVALID_ARGUMENT;
  }
  if (n == 0) {
    set_error("point cloud is empty");
    return CM_EMPTY_CLOUD;
  }
  if (!xyz) {
    set_error("null point pointer");
    return CM_INVALID_ARGUMENT;
  }
  cm_build_options o;
  cm_default_options(&o);
  o.flavor = CM_SPARSE;
  o.mode = CM_TWOD;
  cm_index* ix = nullptr;
  CM_TRY(cm_build(xyz, n, &o, device, stream, &ix));
  DeviceGuard dg(device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  struct Cleanup {
    cm_index* ix;
    std::vector<void*> bufs;
    cudaStream_t st;
    ~Cleanup() {
      for (void* p : bufs) dev_free(p, st);
      cudaStreamSynchronize(st);
      cm_free(ix);
    }
  } cl{ix, {}, st};
  InBuf in;
  CM_TRY(stage_input(xyz, n * 24, st, &in));
  const double* qd = static_cast<const double*>(in.dev);
  uint64_t nq = n;
  if (sample_size && sample_size < n) {
    std::vector<uint64_t> sample(n);
    for (uint64_t i = 0; i < n; ++i) sample[i] = i;
    std::mt19937_64 eng(seed);
    for (uint64_t i = 0; i < sample_size; ++i) {
      const uint64_t j = i + eng() % (sample.size() - i);
      std::swap(sample[i], sample[j]);
    }
    nq = sample_size;
    uint64_t* didx = nullptr;
    double* dq = nullptr;
    CM_CUDA_TRY(dev_alloc_t(&didx, nq, st));
    cl.bufs.push_back(didx);
    CM_CUDA_TRY(dev_alloc_t(&dq, nq * 3, st));
    cl.bufs.push_back(dq);
    CM_CUDA_TRY(cudaMemcpyAsync(didx, sample.data(), nq * 8, cudaMemcpyHostToDevice, st));
    CM_TRY(gather_points_dev(qd, didx, nq, dq, st));
    CM_CUDA_TRY(cudaStreamSynchronize(st));  // `sample` goes out of scope
    qd = dq;
  }
  uint32_t* counts = nullptr;
  unsigned long long* bins = nullptr;
  CM_CUDA_TRY(dev_alloc_t(&counts, nq, st));
  cl.bufs.push_back(counts);
  CM_CUDA_TRY(dev_alloc_t(&bins, 256, st));
  cl.bufs.push_back(bins);
  QueryOrder ord;
  CM_TRY(order_queries(ix, qd, nq, st, &ord, 1.0, CM_CYLINDER));
  CM_TRY(radius_count_dev(ix, qd, nq, CM_CYLINDER, 1.0, ord.perm, counts, nullptr, st));
  CM_TRY(density_histogram_dev(counts, nq, bins, st));
  unsigned long long hb[256];
  CM_CUDA_TRY(cudaMemcpyAsync(hb, bins, sizeof(hb), cudaMemcpyDeviceToHost, st));
  CM_CUDA_TRY(cudaStreamSynchronize(st));
  uint64_t ws = 0, tot = 0;
  for (int b = 0; b < 256; ++b) {
    bins256[b] = hb[b];
    ws += (uint64_t)b * hb[b];
    tot += hb[b];
  }
  *value = static_cast<double>(ws) / static_cast<double>(tot);
  return CM_OK;
}

cm_status cm_knn(const cm_index* ix, const double* q, uint64_t nq, uint32_t k, uint32_t* idx,
                 double* d2, void* stream) {
  CM_TRY(check_index(ix));
  if (k == 0) {  // search.cpp:90-92
    set_error("k must be at least 1");
    return CM_INVALID_ARGUMENT;
  }
  if (nq && (!q || !idx)) {
    set_error("null query or output pointer");
    return CM_INVALID_ARGUMENT;
  }
  DeviceGuard dg(ix->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  InBuf in;
  CM_TRY(stage_input(q, nq * 24, st, &in));
  OutBuf<uint32_t> oi;
  OutBuf<double> od;
  CM_TRY(oi.init(idx, nq * k, st));
  CM_TRY(od.init(d2, nq * k, st));
  QueryOrder ord;
  // 2D Morton centre order: measured no change for config 3 (the tile
  // hulls are set by the centre density, not the curve); opt-in
  static const bool morton = std::getenv("CMGPU_KNN_MORTON") != nullptr;
  CM_TRY(order_queries(ix, static_cast<const double*>(in.dev), nq, st, &ord, -1.0, 0, morton));
  CM_TRY(knn_dev(ix, static_cast<const double*>(in.dev), nq, k, ord.perm, oi.dev, od.dev, st));
  CM_TRY(oi.finish());
  CM_TRY(od.finish());
  return sync_if(oi.host() || od.host(), st);
}

}  // extern "C"
