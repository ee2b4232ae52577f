// Host-side index object and internal entry points shared by the build,
// query and kNN translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "filter.cuh"

struct cm_index {
  int device = 0;
  cm_build_options opts{};
  cmg::DevGrid g{};
  uint64_t n = 0;       // points
  uint64_t V = 0;       // total voxels
  uint64_t U = 0;       // non-empty voxels
  uint64_t C = 0;       // non-empty (i, j) columns
  int key_bits = 0;

  cmg::PointRec* rec = nullptr;  // n, cell order
  cmg::FRec* frec = nullptr;     // n, cell order: float records (filter.cuh)
  uint32_t* ids = nullptr;       // n, cell order: handles (rec[].id)
  uint64_t* ukey = nullptr;      // U unique voxel keys (ascending)
  uint32_t* ustart = nullptr;    // U + 1 record offsets
  uint32_t* uk_k = nullptr;      // U voxel z index
  // dense
  uint32_t* dense_off = nullptr;  // V + 1
  // sparse
  cmg::HashSlot* vhash = nullptr;
  uint64_t vmask = 0;
  // mixed
  uint32_t* col_dense = nullptr;  // nx*ny (when the footprint is dense)
  cmg::HashSlot* chash = nullptr;
  uint64_t cmask = 0;
  uint32_t* col_vbeg = nullptr;   // C + 1

  std::vector<uint64_t> slice_ne;  // per z slice non-empty voxels (host)
  // Running estimate of neighbours per query, sizing the single-pass arena.
  // Queries may run concurrently from many host threads (map.hpp:50-52), so
  // it is an atomic; lost updates between threads only change arena sizing.
  mutable std::atomic<double> nnz_per_query{64.0};
  cm_build_timing timing{};
  // handles are global ids of a multi-GPU slab (cm_build_slab), not
  // positions in the indexed points: self queries do not apply
  bool global_ids = false;
  // lazily built (first kNN): handle -> record position, n entries
  mutable uint32_t* rec_of = nullptr;
  mutable std::mutex lazy_mu;

  cmg::Tables tables() const {
    cmg::Tables t{};
    t.g = g;
    t.rec = rec;
    t.frec = frec;
    t.ids = ids;
    t.n = n;
    t.flavor = opts.flavor;
    t.dense_off = dense_off;
    t.vhash = vhash;
    t.vmask = vmask;
    t.col_dense = col_dense;
    t.chash = chash;
    t.cmask = cmask;
    t.col_vbeg = col_vbeg;
    t.uk_k = uk_k;
    t.ustart = ustart;
    return t;
  }
};

namespace cmg {

constexpr int kMaxDevices = 64;

// One T per host thread AND per device: CUDA events and streams belong to
// the device that was current when they were created, and an index may be
// queried from any thread, one device after another. Callers have already
// made the index's device current (DeviceGuard).
template <typename T>
T& per_thread_device() {
  thread_local T* objs[kMaxDevices] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) dev = 0;
  if (!objs[dev]) objs[dev] = new T();
  return *objs[dev];
}

// Device-memory helpers (stream-ordered pool).
cudaError_t dev_alloc(void** p, size_t bytes, cudaStream_t st);
void dev_free(void* p, cudaStream_t st);

template <typename T>
inline cudaError_t dev_alloc_t(T** p, size_t count, cudaStream_t st) {
  return dev_alloc(reinterpret_cast<void**>(p), count * sizeof(T), st);
}

bool is_device_ptr(const void* p);

// A buffer that is the caller's device pointer, or a device copy of a host
// input (freed on destruction).
struct InBuf {
  const void* dev = nullptr;
  void* owned = nullptr;
  cudaStream_t st = nullptr;
  ~InBuf() {
    if (owned) dev_free(owned, st);
  }
};
cm_status stage_input(const void* p, size_t bytes, cudaStream_t st, InBuf* out);

cm_status bbox_dev(const double* xyz, uint64_t n, cudaStream_t st, double lo[3], double hi[3],
                   cudaEvent_t after = nullptr);
cm_status build_index(const double* xyz_dev, uint64_t n, const cm_build_options& o,
                      cudaStream_t st, cm_index* ix, const double* bounds6 = nullptr);

// Query pipeline pieces (query.cu)
struct QueryOrder {
  uint32_t* perm = nullptr;  // sorted position -> query index
  // the centres the kernels read: the caller's, a materialised copy
  // (owned_q), or null = self queries read from the index's records
  const double* q = nullptr;
  double* owned_q = nullptr;
  uint64_t nq = 0;
  cudaStream_t st = nullptr;
  ~QueryOrder() {
    if (perm) dev_free(perm, st);
    if (owned_q) dev_free(owned_q, st);
  }
};
// q_dev == nullptr: self queries (the index's own n points, row q = point q).
// morton: 2D Morton order of the centres' columns (sparse centre sets, kNN)
cm_status order_queries(const cm_index* ix, const double* q_dev, uint64_t nq, cudaStream_t st,
                        QueryOrder* out, double r = -1.0, int kind = 0, bool morton = false);
cm_status radius_count_dev(const cm_index* ix, const double* q_dev, uint64_t nq, int kernel,
                           double r, const uint32_t* perm, uint32_t* counts_dev,
                           uint64_t* tested_dev, cudaStream_t st, const double* rq = nullptr,
                           const double* qbox = nullptr);
bool radius_is_wide(const cm_index* ix, double r);
// brute-force baselines (brute.cu): every point against every centre
constexpr int kBruteKMax = 64;
cm_status csr_digest_dev(const uint64_t* row_ptr, const uint32_t* cols, uint64_t nq,
                         uint32_t* counts, uint64_t* digests, unsigned long long* unsorted,
                         cudaStream_t st);
cm_status brute_radius_dev(const double* xyz, uint64_t n, const double* q, uint64_t nq, int kind,
                           double r, uint32_t* counts, uint64_t* digests, cudaStream_t st);
cm_status brute_knn_dev(const double* xyz, uint64_t n, const double* q, uint64_t nq, uint32_t k,
                        uint32_t* idx, double* d2, cudaStream_t st);
cm_status radius_fill_dev(const cm_index* ix, const double* q_dev, uint64_t nq, int kernel,
                          double r, const uint32_t* perm, const uint64_t* row_ptr_dev,
                          uint32_t* cols_dev, cudaStream_t st, cudaEvent_t after_fill = nullptr,
                          uint32_t mid_min = 0, const double* rq = nullptr,
                          const double* qbox = nullptr);
cm_status row_class_counts_dev(const uint32_t* counts, uint64_t nq, unsigned long long* out,
                               cudaStream_t st);
cm_status radius_digest_dev(const cm_index* ix, const double* q_dev, uint64_t nq, int kernel,
                            double r, const uint32_t* perm, uint32_t* counts_dev,
                            uint64_t* digest_dev, cudaStream_t st, const double* rq = nullptr,
                            const double* qbox = nullptr);
// Long COLLECT rows (one query per warp, > kSortCap handles), left in visit
// order for merge_big_rows: arena offset, length and query of each.
struct MergeList {
  uint64_t* off = nullptr;
  uint32_t* len = nullptr;
  uint32_t* q = nullptr;
  uint32_t* n = nullptr;
  cudaStream_t st = nullptr;
  ~MergeList() {
    if (off) dev_free(off, st);
    if (len) dev_free(len, st);
    if (q) dev_free(q, st);
    if (n) dev_free(n, st);
  }
};
uint32_t long_row_min();
cm_status merge_big_rows(const MergeList& ml, uint32_t* arena, const uint64_t* row_ptr,
                         uint32_t* cols, cudaStream_t st);
cm_status radius_collect_dev(const cm_index* ix, const double* q_dev, uint64_t nq, int kernel,
                             double r, const uint32_t* perm, uint32_t* temp, uint64_t cap,
                             uint64_t* toff, uint32_t* scnt, uint32_t* counts,
                             unsigned long long* cursor, cudaStream_t st,
                             cudaEvent_t after_collect, const double* rq = nullptr,
                             const double* qbox = nullptr, const MergeList* ml = nullptr);
cm_status gather_rows_dev(const uint32_t* temp, const uint64_t* toff, const uint32_t* scnt,
                          const uint64_t* row_ptr, const uint32_t* perm, uint32_t* cols,
                          uint64_t nq, cudaStream_t st, uint32_t skip_above = 0xffffffffu);
cm_status counts_to_row_ptr(const uint32_t* counts_dev, uint64_t nq, uint64_t* row_ptr_dev,
                            cudaStream_t st);
cm_status knn_dev(const cm_index* ix, const double* q_dev, uint64_t nq, uint32_t k,
                  const uint32_t* perm, uint32_t* idx_dev, double* d2_dev, cudaStream_t st);

cm_status density_histogram_dev(const uint32_t* counts, uint64_t n, unsigned long long* bins,
                                cudaStream_t st);
cm_status gather_points_dev(const double* xyz, const uint64_t* idx, uint64_t n, double* out,
                            cudaStream_t st);
int sm_count();
void query_stats(uint64_t* out, int reset);

}  // namespace cmg
