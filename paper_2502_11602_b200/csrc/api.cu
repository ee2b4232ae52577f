// C ABI (include/cmgpu.h): argument checks, host/device staging, ownership.
#include <algorithm>
#include <atomic>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "index.cuh"
#include "sort_scan.cuh"

namespace cmg {

namespace {
thread_local std::string g_last_error;
std::mutex g_pool_mu;
bool g_pool_configured[64] = {};
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

static void configure_pool() {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_pool_mu);
  if (dev >= 0 && dev < 64 && !g_pool_configured[dev]) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = ~0ull;  // keep freed blocks cached across calls
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    g_pool_configured[dev] = true;
  }
}

cudaError_t dev_alloc(void** p, size_t bytes, cudaStream_t st) {
  configure_pool();
  return cudaMallocAsync(p, bytes == 0 ? 16 : bytes, st);
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
  if (kernel != CM_SPHERE && kernel != CM_CUBE) {
    set_error("unknown kernel (CM_SPHERE = 0, CM_CUBE = 1)");
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

const char* cm_status_name(cm_status s) {
  switch (s) {
    case CM_OK: return "CM_OK";
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
  void* ptrs[] = {ix->rec,   ix->ukey,  ix->ustart, ix->uk_k,    ix->dense_off,
                  ix->vhash, ix->col_dense, ix->chash, ix->col_vbeg};
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
__global__ void corrupt_kernel(uint32_t* ustart, uint32_t* dense_off, uint64_t first_key,
                               HashSlot* vhash, uint64_t vmask) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (dense_off)
    for (uint64_t g = tid; g <= first_key; g += (uint64_t)gridDim.x * blockDim.x) dense_off[g] = 1;
  if (tid == 0) {
    ustart[0] += 1;
    if (vhash) {
      uint64_t s = mix64(first_key) & vmask;
      while (vhash[s].key != first_key) s = (s + 1) & vmask;
      vhash[s].a += 1;
    }
  }
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

cm_status cm_corrupt_for_testing(cm_index* ix) {
  CM_TRY(check_index(ix));
  DeviceGuard dg(ix->device);
  uint64_t first = 0;
  CM_CUDA_TRY(cudaMemcpy(&first, ix->ukey, 8, cudaMemcpyDeviceToHost));
  apik::corrupt_kernel<<<64, 256, 0, 0>>>(ix->ustart, ix->dense_off, first, ix->vhash, ix->vmask); ::cmg::note_launch();
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
  CM_TRY(order_queries(ix, static_cast<const double*>(in.dev), nq, st, &ord));
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
  CM_TRY(order_queries(ix, static_cast<const double*>(in.dev), nq, st, &ord));
  CM_TRY(radius_fill_dev(ix, static_cast<const double*>(in.dev), nq, kernel, r, ord.perm,
                         static_cast<const uint64_t*>(rp.dev), c.dev, st));
  CM_TRY(c.finish());
  return sync_if(c.host(), st);
}

}  // extern "C"

namespace {
struct QueryEvents {
  cudaEvent_t e[6];
  uint64_t nq = 0, nnz = 0;
  bool two_pass = false;
  bool valid = false;
  QueryEvents() {
    for (auto& x : e) cudaEventCreate(&x);
  }
};
thread_local QueryEvents* g_qev = nullptr;
QueryEvents& qev() {
  if (!g_qev) g_qev = new QueryEvents();
  return *g_qev;
}
}  // namespace

extern "C" {

cm_status cm_get_last_query_timing(cm_query_timing* o) {
  if (!o) return CM_INVALID_ARGUMENT;
  QueryEvents& ev = qev();
  if (!ev.valid) {
    set_error("no radius search has run on this thread");
    return CM_INVALID_ARGUMENT;
  }
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
  o->two_pass = ev.two_pass ? 1 : 0;
  return CM_OK;
}

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
  const double* qd = static_cast<const double*>(in.dev);
  QueryEvents& ev = qev();
  ev.valid = false;
  cudaEventRecord(ev.e[0], st);
  QueryOrder ord;
  CM_TRY(order_queries(ix, qd, nq, st, &ord));
  cudaEventRecord(ev.e[1], st);
  cm_csr* csr = new cm_csr();
  csr->nq = nq;
  csr->device = ix->device;
  uint32_t* counts = nullptr;
  uint64_t* toff = nullptr;
  uint32_t* temp = nullptr;
  unsigned long long* cursor = nullptr;
  auto release = [&]() {
    if (counts) dev_free(counts, st);
    if (toff) dev_free(toff, st);
    if (temp) dev_free(temp, st);
    if (cursor) dev_free(cursor, st);
    counts = nullptr, toff = nullptr, temp = nullptr, cursor = nullptr;
  };
  auto fail = [&](cm_status s) {
    release();
    cudaStreamSynchronize(st);
    cm_csr_free(csr);
    return s;
  };
  if (dev_alloc_t(&counts, nq + 1, st) != cudaSuccess ||
      dev_alloc_t(&csr->row_ptr, nq + 1, st) != cudaSuccess ||
      dev_alloc_t(&toff, nq + 1, st) != cudaSuccess || dev_alloc_t(&cursor, 1, st) != cudaSuccess) {
    set_error("device allocation failed (row pointers)");
    return fail(CM_CUDA);
  }
  // Single pass: sorted rows into an arena sized from the running
  // neighbours-per-query estimate; if the arena overflows, fall back to
  // count + scan + fill.
  uint64_t cap = (uint64_t)((double)nq * ix->nnz_per_query * 1.05) + (1u << 20);
  bool two_pass = dev_alloc_t(&temp, cap, st) != cudaSuccess;
  if (two_pass) cudaGetLastError();
  cm_status s = CM_OK;
  unsigned long long used = 0;
  if (!two_pass) {
    s = radius_collect_dev(ix, qd, nq, kernel, r, ord.perm, temp, cap, toff, counts, cursor, st,
                           ev.e[2]);
    cudaEventRecord(ev.e[3], st);
    if (s != CM_OK) return fail(s);
    if (cudaMemcpyAsync(&used, cursor, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess) {
      set_error("arena cursor readback failed");
      return fail(CM_CUDA);
    }
    if (nq) ix->nnz_per_query = std::max(1.0, (double)used / (double)nq);
    two_pass = used > cap;
    if (two_pass) {
      dev_free(temp, st);
      temp = nullptr;
    }
  }
  if (two_pass) {
    cudaEventRecord(ev.e[1], st);
    s = radius_count_dev(ix, qd, nq, kernel, r, ord.perm, counts, nullptr, st);
    cudaEventRecord(ev.e[2], st);
    cudaEventRecord(ev.e[3], st);
    if (s != CM_OK) return fail(s);
  }
  s = counts_to_row_ptr(counts, nq, csr->row_ptr, st);
  cudaEventRecord(ev.e[4], st);
  if (s != CM_OK) return fail(s);
  if (two_pass) {
    if (cudaMemcpyAsync(&csr->nnz, csr->row_ptr + nq, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess) {
      set_error("row pointer readback failed");
      return fail(CM_CUDA);
    }
  } else {
    csr->nnz = used;
  }
  if (dev_alloc_t(&csr->cols, csr->nnz, st) != cudaSuccess) {
    set_error("device allocation failed (columns)");
    return fail(CM_CUDA);
  }
  if (two_pass)
    s = radius_fill_dev(ix, qd, nq, kernel, r, ord.perm, csr->row_ptr, csr->cols, st, nullptr);
  else
    s = gather_rows_dev(temp, toff, counts, csr->row_ptr, csr->cols, nq, st);
  cudaEventRecord(ev.e[5], st);
  if (s != CM_OK) return fail(s);
  ev.nq = nq;
  ev.nnz = csr->nnz;
  ev.two_pass = two_pass;
  ev.valid = true;
  release();
  *out = csr;
  return CM_OK;
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
  CM_TRY(order_queries(ix, static_cast<const double*>(in.dev), nq, st, &ord));
  CM_TRY(radius_digest_dev(ix, static_cast<const double*>(in.dev), nq, kernel, r, ord.perm, c.dev,
                           d.dev, st));
  CM_TRY(c.finish());
  CM_TRY(d.finish());
  return sync_if(c.host() || d.host(), st);
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
  CM_TRY(order_queries(ix, static_cast<const double*>(in.dev), nq, st, &ord));
  CM_TRY(knn_dev(ix, static_cast<const double*>(in.dev), nq, k, ord.perm, oi.dev, od.dev, st));
  CM_TRY(oi.finish());
  CM_TRY(od.finish());
  return sync_if(oi.host() || od.host(), st);
}

}  // extern "C"
