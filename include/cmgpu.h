/* cmgpu.h — C ABI of the B200 cheesemap cell index and neighbour-query engine.
 *
 * This is the drop-in boundary for the reference's C++ index API
 * (/root/reference/proj/core/include/cheesemap/):
 *
 *   reference                                         replaced by
 *   ------------------------------------------------  -----------------------------
 *   Cheesemap::build(cloud, BuildOptions)  map.hpp:55  cm_build
 *   Cheesemap::grid()                      map.hpp:57  cm_get_grid
 *   Cheesemap::occupancy_stats()     map.hpp:104, map.cpp:150-171  cm_get_occupancy
 *   Cheesemap::memory_report()       map.hpp:105, map.cpp:173-192  cm_get_memory_report
 *   read_las(path)                   io.hpp:39-42, io.cpp:33-106  cm_las_read / cm_las_decode
 *   brute_radius / brute_knn         baseline.hpp:11-21, baseline.cpp:8-25
 *                                                          cm_brute_radius / cm_brute_knn
 *   Cheesemap::voxel_lookup / for_each_in_voxel  map.hpp:69-102  cm_export_voxels
 *   kernel_search<SphereKernel|BoxKernel>  search.hpp:102-127
 *                                 cm_radius_count + cm_radius_fill, cm_radius_search,
 *                                 cm_radius_digest (batched; one row per query centre)
 *   knn_search(map, c, k)                  search.hpp:131-134, search.cpp:87-146
 *                                                               cm_knn (batched)
 *   Cheesemap::corrupt_for_testing()       map.hpp:109, map.cpp:194-223
 *                                                               cm_corrupt_for_testing
 *   cheesemap::Error hierarchy             errors.hpp:8-42     cm_status + cm_last_error
 *
 * The reference has no batch entry point: one C++ call answers one query.
 * Here one call answers a batch; row q of the output is what the reference's
 * call returns for centre q, as a list SORTED ASCENDING (the reference
 * returns visit order; its own tests compare sorted copies,
 * tests/test_util.hpp:30-35).
 *
 * Conventions
 *  - Points are the reference's PointCloud layout (geometry.hpp:13-24):
 *    n x 3 doubles, AoS (x, y, z). A handle is the point's position in that
 *    array (u64 in the reference; u32 here, so n < 2^32).
 *  - Input/output pointers may be HOST or DEVICE memory (detected with
 *    cudaPointerGetAttributes). Host inputs are copied in, host outputs are
 *    copied back and the call synchronises. With device outputs calls are
 *    ordered on `stream` (a cudaStream_t; NULL = legacy default stream);
 *    ordered, not asynchronous: cm_radius_search waits on the host once
 *    inside the call (the arena cursor is read back to size the CSR), so
 *    overlap other work from other host threads.
 *  - A built index is immutable and may be queried concurrently from many
 *    host threads / streams (map.hpp:50-52). The index owns device copies of
 *    the points; the caller's cloud need not outlive it.
 *  - Errors: cm_status with the reference's trigger conditions checked in the
 *    reference's order (map.cpp:23-39, grid.cpp:18-27 and :51-59,
 *    search.cpp:90-92). cm_last_error() returns a thread-local message.
 */
#ifndef CMGPU_H
#define CMGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  CM_OK = 0,
  CM_EMPTY_CLOUD = 1,      /* EmptyCloudError      errors.hpp:13-17 */
  CM_INVALID_ARGUMENT = 2, /* InvalidArgumentError errors.hpp:34-37 */
  CM_CAPACITY = 3,         /* CapacityError        errors.hpp:19-22 */
  CM_OUT_OF_DOMAIN = 4,    /* OutOfDomainError     errors.hpp:24-27 */
  CM_CUDA = 5,             /* CUDA runtime failure (no reference analogue) */
  CM_NCCL = 6,             /* collective failure (multi-GPU slabs) */
  CM_PARSE = 7,            /* ParseError           errors.hpp:29-32 */
  CM_IO = 8                /* IoError              errors.hpp:39-42 */
} cm_status;

/* map.hpp:15 */
typedef enum { CM_DENSE = 0, CM_SPARSE = 1, CM_MIXED = 2 } cm_flavor;
/* grid.hpp:10 */
typedef enum { CM_TWOD = 0, CM_THREED = 1 } cm_grid_mode;
/* geometry.hpp:73-113: SphereKernel{c, r}; BoxKernel{{c-r}, {c+r}} (the cube
 * the reference CLI/tests build, cmd_bench.cpp:107-111); CylinderKernel
 * {c.x, c.y, r} with the default unbounded z range (the kernel
 * weighted_density uses, analysis.cpp:55-59; c.z is ignored) */
typedef enum { CM_SPHERE = 0, CM_CUBE = 1, CM_CYLINDER = 2 } cm_kernel;

/* BuildOptions, field for field (map.hpp:17-26). `reorder` is accepted and
 * ignored: the device index is always stored in cell order, and results are
 * always original handles (what reorder=true returns, map.hpp:131-138). */
typedef struct {
  int32_t flavor;             /* cm_flavor, default CM_DENSE */
  int32_t mode;               /* cm_grid_mode, default CM_THREED */
  double cell_x, cell_y, cell_z; /* default 1.0 */
  int32_t reorder;            /* default 0 */
  double densify_threshold;   /* default 0.80 */
  uint64_t dense_voxel_cap;   /* default 2^32 */
} cm_build_options;

/* GridParams (grid.hpp:47-81) */
typedef struct {
  double origin[3];
  double cell[3];
  uint64_t nx, ny, nz;
  int32_t mode;
  double bounds_min[3], bounds_max[3];
} cm_grid_params;

/* OccupancyStats (map.hpp:34-39); slices are reported for every flavour,
 * with the mixed flavour's densify rule (map.cpp:106-108) applied. */
typedef struct {
  uint64_t total_voxels;
  uint64_t non_empty;
  double empty_fraction;
  uint64_t n_slices;
  uint64_t n_columns;   /* non-empty (i, j) columns (mixed layout) */
} cm_occupancy;

/* Device-side build timing, milliseconds (CUDA events). */
typedef struct {
  double total_ms;      /* device-resident points -> ready index */
  double h2d_ms;        /* host->device copy of the cloud (0 for device input) */
  double bbox_ms, keys_ms, sort_ms, gather_ms, tables_ms;
  uint32_t sort_passes;
} cm_build_timing;

/* Device timing of the last radius call on this host thread (CUDA events on
 * the call's stream), milliseconds. */
typedef struct {
  double order_ms;    /* query cell keys + radix sort (spatial order) */
  double pass1_ms;    /* single pass: collect kernel (sorted rows -> arena);
                         two-pass fallback: count kernel */
  double rowsort_ms;  /* block sort of rows longer than a warp buffer */
  double scan_ms;     /* row_ptr scan */
  double pass2_ms;    /* single pass: gather arena -> CSR; two-pass: fill */
  double total_ms;
  uint64_t nq, nnz;
  int32_t two_pass;   /* 1: count + fill ran (large radius, or no arena); 2: the arena
                         overflowed and the collect reran into one of the exact size */
} cm_query_timing;

typedef struct cm_index cm_index;
typedef struct cm_csr cm_csr;

void cm_default_options(cm_build_options* opts);

/* Cheesemap::build (map.cpp:22-122). xyz: n x 3 doubles, host or device. */
cm_status cm_build(const double* xyz, uint64_t n, const cm_build_options* opts,
                   int device, void* stream, cm_index** out);
/* As cm_build, on the grid of an explicit bounding box instead of the
 * cloud's own (grid_dims(box), grid.cpp:41-61). Used by x-slab partitions so
 * every slab indexes on the global grid; a point outside the box is
 * CM_OUT_OF_DOMAIN (voxel_of, grid.cpp:64-66). */
cm_status cm_build_in_bounds(const double* xyz, uint64_t n, const cm_build_options* opts,
                             const double* bounds_min, const double* bounds_max, int device,
                             void* stream, cm_index** out);
cm_status cm_free(cm_index* index);

cm_status cm_get_grid(const cm_index* index, cm_grid_params* out);
/* Cheesemap::memory_report (map.hpp:41-48, map.cpp:173-192): the
 * reference's analytic byte model for this flavour and occupancy
 * (handle / structure / total bytes), plus device_bytes, the HBM this index
 * actually holds (records + tables). */
typedef struct {
  uint64_t handle_bytes;
  uint64_t structure_bytes;
  uint64_t total_bytes;
  uint64_t device_bytes;
} cm_memory_report;
cm_status cm_get_memory_report(const cm_index* index, cm_memory_report* out);

cm_status cm_get_occupancy(const cm_index* index, cm_occupancy* out,
                           uint8_t* slice_dense, uint64_t* slice_non_empty,
                           uint64_t slice_capacity);
cm_status cm_get_build_timing(const cm_index* index, cm_build_timing* out);
/* Per-voxel handle sets in stored order (key ascending, handles ascending
 * inside a voxel): keys[p], handles[p] for p < n. Host or device outputs. */
cm_status cm_export_voxels(const cm_index* index, uint64_t* keys, uint32_t* handles);
uint64_t cm_size(const cm_index* index);

/* kernel_search, count pass: counts[q] = |result(q)|; optional
 * points_tested[q] = the reference's QueryStats::points_tested
 * (search.hpp:116). Either output may be NULL. */
cm_status cm_radius_count(const cm_index* index, const double* q, uint64_t nq,
                          int kernel, double r, uint32_t* counts,
                          uint64_t* points_tested, void* stream);
/* kernel_search, fill pass: cols[row_ptr[q] .. row_ptr[q+1]) = sorted
 * handles of result(q). row_ptr must come from the counts of the same call
 * arguments (exclusive scan, nq + 1 entries). */
cm_status cm_radius_fill(const cm_index* index, const double* q, uint64_t nq,
                         int kernel, double r, const uint64_t* row_ptr,
                         uint32_t* cols, void* stream);
/* count + scan + fill in one call; the CSR lives in device memory owned by
 * the returned cm_csr. The output size is data-dependent, so this call waits
 * (host-side) for the neighbour total before it allocates the columns; the
 * kernels themselves run in order on `stream`. */
cm_status cm_radius_search(const cm_index* index, const double* q, uint64_t nq,
                           int kernel, double r, void* stream, cm_csr** out);
/* cm_radius_search with every indexed point as a centre (row q = point q):
 * the "every point is a query" workload. Centres are read from the index's
 * own cell-ordered copy of the points, so no query sort runs. */
cm_status cm_radius_search_self(const cm_index* index, int kernel, double r, void* stream,
                                cm_csr** out);
/* The same search with HOST buffers end to end: queries from host memory,
 * the sorted CSR to host memory (row_ptr: nq + 1 entries; cols: up to
 * cols_capacity). With CMGPU_CHUNKS=K in the environment, queries are
 * processed in K chunks on three streams so the host->device copy of chunk
 * i+1 and the device->host copy of chunk i-1 overlap chunk i's kernels (use
 * pinned host buffers); worthwhile only for spatially coherent query order.
 * *nnz_out = total neighbours; CM_CAPACITY if cols_capacity was too small
 * (nothing past the capacity is written). Synchronous. */
cm_status cm_radius_search_to_host(const cm_index* index, const double* q_host, uint64_t nq,
                                   int kernel, double r, uint64_t* row_ptr_host,
                                   uint32_t* cols_host, uint64_t cols_capacity,
                                   uint64_t* nnz_out, void* stream);
cm_status cm_csr_info(const cm_csr* csr, uint64_t* nq, uint64_t* nnz,
                      const uint64_t** row_ptr_device, const uint32_t** cols_device);
/* row_ptr (nq + 1) and cols (nnz) to caller memory (host or device). */
cm_status cm_csr_download(const cm_csr* csr, uint64_t* row_ptr, uint32_t* cols,
                          void* stream);
cm_status cm_csr_free(cm_csr* csr);
/* Verification of a CSR in DEVICE memory: per-row count and digest exactly
 * as cm_radius_digest reports them (either output may be null), and the
 * number of rows that are not strictly ascending (host *unsorted_rows).
 * Synchronous. */
cm_status cm_csr_digest(const uint64_t* row_ptr, const uint32_t* cols, uint64_t nq,
                        uint32_t* counts, uint64_t* digests, uint64_t* unsorted_rows,
                        void* stream);
/* Per-query count and set digest sum(mix64(handle)) mod 2^64 (splitmix64
 * finaliser) — verification of outputs too large to materialise. */
cm_status cm_radius_digest(const cm_index* index, const double* q, uint64_t nq,
                           int kernel, double r, uint32_t* counts,
                           uint64_t* digests, void* stream);

/* kernel_search for a batch of EXPLICIT kernels (geometry.hpp:73-113), each
 * with its own parameters, params = nq rows of:
 *   CM_SPHERE   4 doubles  cx cy cz r           SphereKernel{c, r}
 *   CM_CUBE     6 doubles  min xyz, max xyz     BoxKernel{Aabb} (any box)
 *   CM_CYLINDER 5 doubles  cx cy r z_lo z_hi    CylinderKernel (+-inf: unbounded)
 * Host or device params; sorted rows as cm_radius_search. */
cm_status cm_kernel_search(const cm_index* index, int kernel, const double* params, uint64_t nq,
                           void* stream, cm_csr** out);
/* Counts and QueryStats (search.hpp:12-17) of explicit kernels: counts[q],
 * points_tested[q] and voxels_visited[q] (the voxels of the clamped range,
 * search.hpp:116-119). Any output may be NULL; host or device outputs. */
cm_status cm_kernel_count(const cm_index* index, int kernel, const double* params, uint64_t nq,
                          uint32_t* counts, uint64_t* points_tested, uint64_t* voxels_visited,
                          void* stream);
/* Cheesemap::voxel_present / voxel_lookup (map.hpp:62-69): whether voxel
 * (i, j, k) is materialized (dense flavour: always; mixed: every cell of a
 * densified slice; else non-empty), its handles ascending (up to capacity;
 * host or device) and their number. CM_OUT_OF_DOMAIN outside the grid. */
cm_status cm_voxel_lookup(const cm_index* index, uint64_t i, uint64_t j, uint64_t k, int* present,
                          uint32_t* handles, uint64_t capacity, uint64_t* count);

/* knn_search (search.cpp:87-146), exact, rows ordered by (fp64 squared
 * distance, handle). idx[q*k + t], d2[q*k + t] (d2 may be NULL). Rows of a
 * cloud with fewer than k points are padded with UINT32_MAX / +inf. */
cm_status cm_knn(const cm_index* index, const double* q, uint64_t nq, uint32_t k,
                 uint32_t* idx, double* d2, void* stream);

/* Dataset density metrics (analysis.hpp:17-35), the cylinder-kernel caller
 * of the index.
 * global_density (analysis.cpp:17-24): points per m^2 of the xy bounding
 * rectangle; CM_INVALID_ARGUMENT for a zero-area rectangle.
 * weighted_density (analysis.cpp:26-86): over all points (sample_size = 0)
 * or a seeded subsample (the reference's partial Fisher-Yates with
 * mt19937_64(seed)), count the points in a vertical 1 m cylinder (2D sparse
 * map, 1 m cells), bin count/pi into bins256[256] (last bin clamps) and
 * return the histogram-weighted mean bin in *value. Synchronous. */
cm_status cm_global_density(const double* xyz, uint64_t n, int device, void* stream,
                            double* value);
cm_status cm_weighted_density(const double* xyz, uint64_t n, uint64_t sample_size, uint64_t seed,
                              int device, void* stream, double* value, uint64_t* bins256);

/* Test hook (map.cpp:194-223): drops one stored handle from the first
 * non-empty voxel so verification harnesses can prove they detect it. */
cm_status cm_corrupt_for_testing(cm_index* index);

/* Timing of the last cm_radius_search on this thread (waits for it). */
cm_status cm_get_last_query_timing(cm_query_timing* out);
/* Kernels launched by this library since load (all threads). */
uint64_t cm_launch_count(void);
/* Query-tile counters since the last reset (all zero unless the library is
 * the checked build, libcmgpu_checked.so: the counters cost the wide-tile
 * passes half their speed), count pass then fill pass:
 * tiles, tiles answered one query per warp (fallback), hull points,
 * in-range candidates (count pass only). out8 has 8 entries. */
cm_status cm_debug_query_stats(uint64_t* out8, int reset);
/* The library allocates from a private stream-ordered pool per device.
 * Defaults: nothing reserved up front; large requests grow the pool in
 * blocks of four times the request (CMGPU_POOL_GROW), up to 1/8 of HBM, which
 * is also what stays cached across synchronisations. A process that owns the GPU may keep more cached
 * (keep_bytes) and reserve a block up front (reserve_bytes), so later calls
 * carve from it instead of mapping fresh memory. */
cm_status cm_pool_configure(int device, uint64_t keep_bytes, uint64_t reserve_bytes);
/* Device memory held by this library's stream-ordered pool on `device`:
 * reserved (cached + in use) and in use, in bytes; trim != 0 first returns
 * the cached part to the device. */
cm_status cm_debug_pool_bytes(int device, int trim, uint64_t* reserved, uint64_t* used);

/* ---- brute-force baselines: brute_radius (baseline.hpp:11-21), brute_knn
 * (baseline.cpp:8-25) — every point against every centre, no index; what the
 * CLI's verify compares the index against. brute_radius reports each set as
 * (count, sum of splitmix64(handle)) like cm_radius_digest; brute_knn orders
 * by (d², handle), k <= 64. Points / centres / outputs host or device. */
cm_status cm_brute_radius(const double* xyz, uint64_t n, const double* centers, uint64_t nq,
                          int kernel, double r, uint32_t* counts, uint64_t* digests, int device,
                          void* stream);
cm_status cm_brute_knn(const double* xyz, uint64_t n, const double* centers, uint64_t nq,
                       uint32_t k, uint32_t* idx, double* d2, int device, void* stream);

/* ---- LAS ingestion: read_las (io.hpp:39-42, io.cpp:33-106) ----------------
 * The header is checked on the host with the reference's checks, messages
 * and order (CM_PARSE = ParseError, CM_IO = IoError); the point records are
 * decoded on the device, coordinate = raw * scale + offset in fp64 without
 * FMA (io.cpp:97-103). Point formats 0-8, LAS 1.2-1.4 (64-bit 1.4 counts). */
typedef struct {
  uint8_t version_major, version_minor, point_format;
  uint16_t header_size, record_length;
  uint32_t data_offset;
  uint64_t point_count;
  double scale[3], offset[3];
  double bounds_min[3], bounds_max[3];
} cm_las_header;

/* Header of a LAS image in HOST memory (io.cpp:38-89 checks). */
cm_status cm_las_parse_header(const void* bytes, uint64_t nbytes, cm_las_header* out);
/* Decodes a whole LAS image (host or device memory) into xyz (n x 3 doubles,
 * host or device, capacity in points). xyz == NULL returns the header only.
 * Truncated images fail like the reference (io.cpp:92-96). */
cm_status cm_las_decode(const void* bytes, uint64_t nbytes, double* xyz, uint64_t xyz_capacity,
                        cm_las_header* hdr, int device, void* stream);
/* read_las(path): CM_IO when the file cannot be opened, then cm_las_decode. */
cm_status cm_las_read(const char* path, double* xyz, uint64_t xyz_capacity, cm_las_header* hdr,
                      int device, void* stream);

/* ---- Multi-GPU: x-slabs with a halo ---------------------
 * One rank per GPU (a process, or a host thread). Every rank of a cluster
 * passes ITS share of the cloud (any partition of the points, each with a
 * global id) to cm_build_slab; the ranks then all-reduce the global bounding
 * box (the grid of grid.cpp:41-61 over the whole cloud), cut its x extent
 * into nranks equal slabs, exchange the points so that every rank holds the
 * points of its slab plus the points within `halo` of its faces, and index
 * them on the global grid. A centre owned by a rank then has exactly the
 * neighbour set the single global index gives it, for any r <= halo; rows
 * and digests come out in GLOBAL ids. The map is immutable once built
 * (map.hpp:50-52). Transports: NCCL (the ranks' GPUs, ncclUniqueId from
 * rank 0 passed to every rank by the caller), or in-process (ranks are host
 * threads of one process, e.g. several slabs on one GPU). */
#define CM_CLUSTER_ID_BYTES 128
typedef enum { CM_TRANSPORT_NCCL = 0, CM_TRANSPORT_IN_PROCESS = 1 } cm_transport;
typedef struct cm_cluster cm_cluster;
typedef struct cm_slab cm_slab;
typedef struct {
  double total_ms;    /* device time, device-resident points -> ready slab index,
                         bbox all-reduce and point exchange included */
  double wall_ms;     /* host wall time of the same call */
  double index_ms;    /* of which the local index build */
  uint64_t sent_points, received_points;  /* records packed / received (incl. own) */
} cm_slab_timing;
typedef struct {
  int32_t nranks, rank;
  uint64_t n_local, n_owned, n_halo;
  double halo;
  double bounds[6];   /* global box: min xyz, max xyz */
  cm_slab_timing timing;
} cm_slab_info_t;

/* A fresh group id (CM_CLUSTER_ID_BYTES bytes) for `transport`; rank 0 makes
 * it and the caller hands it to every rank. */
cm_status cm_cluster_unique_id(int transport, void* id_out);
cm_status cm_cluster_init(int transport, const void* id, int nranks, int rank, int device,
                          cm_cluster** out);
cm_status cm_cluster_free(cm_cluster* cluster);
/* Collective over the cluster. xyz: n points (host or device); gids: their
 * global ids (u32, host or device), or NULL for gid_base + i. */
cm_status cm_build_slab(cm_cluster* cluster, const double* xyz, const uint32_t* gids,
                        uint64_t gid_base, uint64_t n, const cm_build_options* opts, double halo,
                        void* stream, cm_slab** out);
cm_status cm_slab_free(cm_slab* slab);
/* edges: nranks + 1 slab boundaries (slab s = [e_s, e_s+1), the last closed) */
cm_status cm_slab_info(const cm_slab* slab, cm_slab_info_t* out, double* edges,
                       uint64_t edges_capacity);
/* The rank's local index (owned + halo points; handles are global ids). */
const cm_index* cm_slab_index(const cm_slab* slab);
/* Owned global ids (n_owned, ascending: the row order of q = NULL queries)
 * and local ones (n_local, ascending); either may be NULL. */
cm_status cm_slab_ids(const cm_slab* slab, uint32_t* owned_gids, uint32_t* local_gids,
                      void* stream);
/* kernel_search for centres inside this slab, r <= halo; q = NULL: every
 * owned point (row i = owned point i). Columns are global ids. */
cm_status cm_slab_radius_search(const cm_slab* slab, const double* q, uint64_t nq, int kernel,
                                double r, void* stream, cm_csr** out);
cm_status cm_slab_radius_digest(const cm_slab* slab, const double* q, uint64_t nq, int kernel,
                                double r, uint32_t* counts, uint64_t* digests, void* stream);

const char* cm_last_error(void);
const char* cm_status_name(cm_status s);

#ifdef __cplusplus
}
#endif

#endif /* CMGPU_H */
