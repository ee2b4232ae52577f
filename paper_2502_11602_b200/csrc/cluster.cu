// Multi-GPU x-slab layout behind the C ABI (include/cmgpu.h
// "Multi-GPU"). One process (or host thread) per GPU; each rank owns the
// points whose x falls in its slab of the GLOBAL bounding box, plus a halo of
// its neighbours' points within `halo` of the shared faces, and indexes them
// on the global grid, so a centre the rank owns sees exactly the candidate
// set of the single global index for any r <= halo.
//
// Reference contracts the layout rests on: the map is immutable and
// concurrently readable (map.hpp:50-52), and the grid is derived from the
// cloud's bounding box (grid.cpp:41-61) — here the all-reduced one, so every
// voxel key and clamped range equals the global index's.
//
// Build (cm_build_slab), every step on the device except two tiny host
// decisions (the global box, the receive sizes):
//   1. local bbox (K1 of the build) -> one MIN all-reduce of (lo, -hi);
//   2. slab edges e_s = lo + (hi - lo) * s / P (the last one = hi);
//   3. classify + pack: each input point goes to its owner slab, and to the
//      neighbour slab whose halo it lies in, as a 32-B record {x, y, z,
//      global id, owned flag} bucketed by destination (one pass counts, one
//      scatters);
//   4. all-to-all of the bucket sizes, then one grouped send/recv of the
//      buckets (NCCL over NVLink, or an in-process transport);
//   5. local records sorted by global id (radix sort), split into the local
//      cloud, the local-handle -> global-id map and the owned centres;
//   6. the local index on the global grid (cm_build_in_bounds' build).
// Local handles ascend with global ids, so sorted local rows stay sorted
// once mapped to global ids.
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <random>
#include <string>
#include <vector>

#include <nccl.h>

#include "index.cuh"
#include "sort_scan.cuh"

namespace cmg {

// ------------------------------------------------------------ transports --
// The collective plumbing of one rank. NCCL for real GPUs; the in-process
// transport runs the same build with ranks as host threads of one process
// (e.g. several ranks on one GPU in tests), copying between device buffers.
struct Transport {
  int P = 1, rank = 0;
  // in/out host v[6]: min over ranks of v[0..6) (callers negate maxima)
  virtual cm_status allreduce_min6(double* v, cudaStream_t st) = 0;
  // host send[P] -> host recv[P]: recv[s] = what rank s sent to this rank
  virtual cm_status alltoall_u64(const uint64_t* send, uint64_t* recv, cudaStream_t st) = 0;
  // device buffers: send[d] (bytes sb[d]) to rank d, recv[s] (rb[s]) from s
  virtual cm_status exchange(const void* const* send, const uint64_t* sb, void* const* recv,
                             const uint64_t* rb, cudaStream_t st) = 0;
  virtual ~Transport() = default;
};

namespace {

// NCCL, loaded at run time: the library itself has no link-time dependency
// on it, and a process that already loaded NCCL (torch) shares that copy.
struct NcclApi {
  bool ok = false;
  std::string err;
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclAllReduce) AllReduce = nullptr;
  decltype(&ncclSend) Send = nullptr;
  decltype(&ncclRecv) Recv = nullptr;
  decltype(&ncclGroupStart) GroupStart = nullptr;
  decltype(&ncclGroupEnd) GroupEnd = nullptr;
  decltype(&ncclGetErrorString) GetErrorString = nullptr;
  NcclApi() {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = std::string("libnccl.so.2 not loadable: ") + dlerror();
      return;
    }
#define CM_NCCL_SYM(name)                                               \
  name = reinterpret_cast<decltype(name)>(dlsym(h, "nccl" #name));      \
  if (!name) {                                                          \
    err = "NCCL symbol nccl" #name " missing";                          \
    return;                                                             \
  }
    CM_NCCL_SYM(GetUniqueId)
    CM_NCCL_SYM(CommInitRank)
    CM_NCCL_SYM(CommDestroy)
    CM_NCCL_SYM(AllReduce)
    CM_NCCL_SYM(Send)
    CM_NCCL_SYM(Recv)
    CM_NCCL_SYM(GroupStart)
    CM_NCCL_SYM(GroupEnd)
    CM_NCCL_SYM(GetErrorString)
#undef CM_NCCL_SYM
    ok = true;
  }
};

NcclApi& nccl() {
  static NcclApi api;
  return api;
}

#define CM_NCCL_TRY(expr)                                                          \
  do {                                                                             \
    ncclResult_t _r = (expr);                                                      \
    if (_r != ncclSuccess) {                                                       \
      set_error(std::string(#expr) + ": " + nccl().GetErrorString(_r));            \
      return CM_NCCL;                                                              \
    }                                                                              \
  } while (0)

struct NcclTransport : Transport {
  ncclComm_t comm = nullptr;
  double* d6 = nullptr;      // device scratch for the all-reduce
  uint64_t* dcnt = nullptr;  // 2P device counters for the all-to-all
  ~NcclTransport() override {
    if (d6) cudaFree(d6);
    if (dcnt) cudaFree(dcnt);
    if (comm) nccl().CommDestroy(comm);
  }
  cm_status allreduce_min6(double* v, cudaStream_t st) override {
    CM_CUDA_TRY(cudaMemcpyAsync(d6, v, 48, cudaMemcpyHostToDevice, st));
    CM_NCCL_TRY(nccl().AllReduce(d6, d6, 6, ncclFloat64, ncclMin, comm, st));
    CM_CUDA_TRY(cudaMemcpyAsync(v, d6, 48, cudaMemcpyDeviceToHost, st));
    CM_CUDA_TRY(cudaStreamSynchronize(st));
    return CM_OK;
  }
  cm_status alltoall_u64(const uint64_t* send, uint64_t* recv, cudaStream_t st) override {
    CM_CUDA_TRY(cudaMemcpyAsync(dcnt, send, 8 * P, cudaMemcpyHostToDevice, st));
    CM_NCCL_TRY(nccl().GroupStart());
    for (int p = 0; p < P; ++p) {
      CM_NCCL_TRY(nccl().Send(dcnt + p, 1, ncclUint64, p, comm, st));
      CM_NCCL_TRY(nccl().Recv(dcnt + P + p, 1, ncclUint64, p, comm, st));
    }
    CM_NCCL_TRY(nccl().GroupEnd());
    CM_CUDA_TRY(cudaMemcpyAsync(recv, dcnt + P, 8 * P, cudaMemcpyDeviceToHost, st));
    CM_CUDA_TRY(cudaStreamSynchronize(st));
    return CM_OK;
  }
  cm_status exchange(const void* const* send, const uint64_t* sb, void* const* recv,
                     const uint64_t* rb, cudaStream_t st) override {
    CM_NCCL_TRY(nccl().GroupStart());
    for (int p = 0; p < P; ++p) {
      if (sb[p]) CM_NCCL_TRY(nccl().Send(send[p], sb[p], ncclChar, p, comm, st));
      if (rb[p]) CM_NCCL_TRY(nccl().Recv(recv[p], rb[p], ncclChar, p, comm, st));
    }
    CM_NCCL_TRY(nccl().GroupEnd());
    return CM_OK;
  }
};

// In-process transport: the ranks of one group are host threads that share
// a mailbox keyed by the group id. Every collective is bracketed by a
// generation barrier, so posted buffers stay valid until all ranks consumed
// them.
struct LocalGroup {
  std::mutex mu;
  std::condition_variable cv;
  int P = 0;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<double> red;
  std::vector<uint64_t> cnt;
  std::vector<const void*> ptr;
  std::vector<uint64_t> bytes;
  explicit LocalGroup(int p) : P(p), red(6 * p), cnt(p * p), ptr(p * p), bytes(p * p) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t g = gen;
    if (++arrived == P) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

std::mutex g_groups_mu;
std::map<std::string, std::weak_ptr<LocalGroup>> g_groups;

struct LocalTransport : Transport {
  std::shared_ptr<LocalGroup> grp;
  cm_status allreduce_min6(double* v, cudaStream_t) override {
    for (int i = 0; i < 6; ++i) grp->red[6 * rank + i] = v[i];
    grp->barrier();
    for (int i = 0; i < 6; ++i) {
      double m = grp->red[i];
      for (int p = 1; p < P; ++p) m = std::min(m, grp->red[6 * p + i]);
      v[i] = m;
    }
    grp->barrier();
    return CM_OK;
  }
  cm_status alltoall_u64(const uint64_t* send, uint64_t* recv, cudaStream_t) override {
    for (int d = 0; d < P; ++d) grp->cnt[rank * P + d] = send[d];
    grp->barrier();
    for (int s = 0; s < P; ++s) recv[s] = grp->cnt[s * P + rank];
    grp->barrier();
    return CM_OK;
  }
  cm_status exchange(const void* const* send, const uint64_t* sb, void* const* recv,
                     const uint64_t* rb, cudaStream_t st) override {
    CM_CUDA_TRY(cudaStreamSynchronize(st));  // the send buffers are complete
    for (int d = 0; d < P; ++d) {
      grp->ptr[rank * P + d] = send[d];
      grp->bytes[rank * P + d] = sb[d];
    }
    grp->barrier();
    cm_status s = CM_OK;
    for (int p = 0; p < P && s == CM_OK; ++p) {
      if (grp->bytes[p * P + rank] != rb[p]) {
        set_error("in-process exchange: size mismatch");
        s = CM_NCCL;
      } else if (rb[p] && cudaMemcpyAsync(recv[p], grp->ptr[p * P + rank], rb[p],
                                          cudaMemcpyDefault, st) != cudaSuccess) {
        set_error("in-process exchange: copy failed");
        s = CM_CUDA;
      }
    }
    if (s == CM_OK && cudaStreamSynchronize(st) != cudaSuccess) s = CM_CUDA;
    grp->barrier();  // every rank has copied out of every send buffer
    return s;
  }
};

// ---------------------------------------------------------------- kernels --
constexpr int kMaxRanks = 64;

struct SlabEdges {
  double e[kMaxRanks + 1];
  int P;
  double halo;
};

// Owner slab of x: the number of inner edges <= x (edges ascending).
__device__ __forceinline__ int owner_of(const SlabEdges& E, double x) {
  int o = 0;
  for (int s = 1; s < E.P; ++s) o += x >= E.e[s];
  return o;
}

// Destinations of a point in slab o: o (owned); o - 1 when it lies within
// the halo above that slab's upper face e[o]; o + 1 within the halo below
// the next slab's lower face e[o + 1].
__device__ __forceinline__ void dests_of(const SlabEdges& E, double x, int* o, bool* dn, bool* up) {
  *o = owner_of(E, x);
  *dn = *o > 0 && x < E.e[*o] + E.halo;
  *up = *o < E.P - 1 && x >= E.e[*o + 1] - E.halo;
}

__global__ void slab_count_kernel(const double* __restrict__ xyz, uint64_t n, SlabEdges E,
                                  unsigned long long* __restrict__ counts) {
  __shared__ unsigned int sc[kMaxRanks];
  for (int i = threadIdx.x; i < E.P; i += blockDim.x) sc[i] = 0;
  __syncthreads();
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < n;
       p += (uint64_t)gridDim.x * blockDim.x) {
    int o;
    bool dn, up;
    dests_of(E, xyz[3 * p], &o, &dn, &up);
    atomicAdd(&sc[o], 1u);
    if (dn) atomicAdd(&sc[o - 1], 1u);
    if (up) atomicAdd(&sc[o + 1], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < E.P; i += blockDim.x)
    if (sc[i]) atomicAdd(&counts[i], (unsigned long long)sc[i]);
}

// Records bucketed by destination; `cursor[d]` starts at bucket d's offset.
// PointRec.k carries the owned flag (1 = the destination owns the point).
__global__ void slab_pack_kernel(const double* __restrict__ xyz, const uint32_t* __restrict__ gids,
                                 uint64_t gid_base, uint64_t n, SlabEdges E,
                                 unsigned long long* __restrict__ cursor,
                                 PointRec* __restrict__ out, uint64_t total) {
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < n;
       p += (uint64_t)gridDim.x * blockDim.x) {
    PointRec r;
    r.x = xyz[3 * p];
    r.y = xyz[3 * p + 1];
    r.z = xyz[3 * p + 2];
    r.id = gids ? gids[p] : (uint32_t)(gid_base + p);
    int o;
    bool dn, up;
    dests_of(E, r.x, &o, &dn, &up);
    r.k = 1;
    const unsigned long long a = atomicAdd(&cursor[o], 1ull);
    CM_DCHECK(a < total);
    out[a] = r;
    r.k = 0;
    if (dn) {
      const unsigned long long b = atomicAdd(&cursor[o - 1], 1ull);
      CM_DCHECK(b < total);
      out[b] = r;
    }
    if (up) {
      const unsigned long long c = atomicAdd(&cursor[o + 1], 1ull);
      CM_DCHECK(c < total);
      out[c] = r;
    }
  }
}

__global__ void slab_keys_kernel(const PointRec* __restrict__ rec, uint64_t n,
                                 uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < n;
       p += (uint64_t)gridDim.x * blockDim.x) {
    keys[p] = rec[p].id;
    vals[p] = (uint32_t)p;
  }
}

// Local cloud in global-id order + handle -> global id map + owned flags.
__global__ void slab_unpack_kernel(const PointRec* __restrict__ rec, const uint32_t* __restrict__ order,
                                   uint64_t n, double* __restrict__ xyz, uint32_t* __restrict__ gid,
                                   uint32_t* __restrict__ owned) {
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < n;
       p += (uint64_t)gridDim.x * blockDim.x) {
    const PointRec r = rec[order[p]];
    xyz[3 * p] = r.x;
    xyz[3 * p + 1] = r.y;
    xyz[3 * p + 2] = r.z;
    gid[p] = r.id;
    owned[p] = r.k;
  }
}

// Owned points (flag 1) compacted in local (= global id) order.
__global__ void slab_owned_kernel(const double* __restrict__ xyz, const uint32_t* __restrict__ gid,
                                  const uint32_t* __restrict__ owned,
                                  const uint32_t* __restrict__ pos, uint64_t n,
                                  double* __restrict__ oxyz, uint32_t* __restrict__ ogid) {
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < n;
       p += (uint64_t)gridDim.x * blockDim.x) {
    if (!owned[p]) continue;
    const uint32_t o = pos[p];
    oxyz[3 * (uint64_t)o] = xyz[3 * p];
    oxyz[3 * (uint64_t)o + 1] = xyz[3 * p + 1];
    oxyz[3 * (uint64_t)o + 2] = xyz[3 * p + 2];
    ogid[o] = gid[p];
  }
}

// After the local build: every record's handle becomes its global id, so
// all query outputs (CSR, digests, kNN, exports) come out in global ids.
// Local handles ascend with global ids, so row order is unchanged.
__global__ void relabel_kernel(PointRec* __restrict__ rec, uint32_t* __restrict__ ids, uint64_t n,
                               const uint32_t* __restrict__ gid) {
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < n;
       p += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t g = __ldg(gid + rec[p].id);
    rec[p].id = g;
    ids[p] = g;
  }
}

unsigned grid_of(uint64_t n) {
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, (uint64_t)sm_count() * 8));
}

}  // namespace
}  // namespace cmg

struct cm_cluster {
  int device = 0;
  std::unique_ptr<cmg::Transport> tr;
};

struct cm_slab {
  cm_cluster* cl = nullptr;
  cm_index* ix = nullptr;        // owned + halo points, global grid (null if none)
  uint32_t* local_gid = nullptr;  // local handle -> global id (ascending)
  double* owned_xyz = nullptr;    // owned centres, global-id order
  uint32_t* owned_gid = nullptr;
  uint64_t n_local = 0, n_owned = 0, n_halo = 0;
  double halo = 0.0;
  double bounds[6] = {0, 0, 0, 0, 0, 0};
  std::vector<double> edges;
  cm_slab_timing timing{};
};

using namespace cmg;

namespace {
struct DevGuard {
  int prev = -1;
  explicit DevGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DevGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};
}  // namespace

extern "C" {

cm_status cm_cluster_unique_id(int transport, void* id_out) {
  if (!id_out) {
    set_error("null id output");
    return CM_INVALID_ARGUMENT;
  }
  std::memset(id_out, 0, CM_CLUSTER_ID_BYTES);
  if (transport == CM_TRANSPORT_NCCL) {
    if (!nccl().ok) {
      set_error(nccl().err);
      return CM_NCCL;
    }
    static_assert(sizeof(ncclUniqueId) <= CM_CLUSTER_ID_BYTES, "ncclUniqueId size");
    ncclUniqueId u;
    CM_NCCL_TRY(nccl().GetUniqueId(&u));
    std::memcpy(id_out, &u, sizeof(u));
    return CM_OK;
  }
  if (transport == CM_TRANSPORT_IN_PROCESS) {
    std::random_device rd;
    uint64_t w[4] = {((uint64_t)rd() << 32) ^ rd(), ((uint64_t)rd() << 32) ^ rd(),
                     (uint64_t)std::chrono::steady_clock::now().time_since_epoch().count(), 0x63686565ull};
    std::memcpy(id_out, w, sizeof(w));
    return CM_OK;
  }
  set_error("unknown transport (CM_TRANSPORT_NCCL = 0, CM_TRANSPORT_IN_PROCESS = 1)");
  return CM_INVALID_ARGUMENT;
}

cm_status cm_cluster_init(int transport, const void* id, int nranks, int rank, int device,
                          cm_cluster** out) {
  if (!out || !id) {
    set_error("null id or output");
    return CM_INVALID_ARGUMENT;
  }
  *out = nullptr;
  if (nranks < 1 || nranks > kMaxRanks || rank < 0 || rank >= nranks) {
    set_error("rank / nranks out of range (1 <= nranks <= 64)");
    return CM_INVALID_ARGUMENT;
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
    cudaGetLastError();
    set_error("device ordinal out of range");
    return CM_INVALID_ARGUMENT;
  }
  DevGuard dg(device);
  auto cl = std::make_unique<cm_cluster>();
  cl->device = device;
  if (transport == CM_TRANSPORT_NCCL) {
    if (!nccl().ok) {
      set_error(nccl().err);
      return CM_NCCL;
    }
    auto t = std::make_unique<NcclTransport>();
    t->P = nranks, t->rank = rank;
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    CM_NCCL_TRY(nccl().CommInitRank(&t->comm, nranks, u, rank));
    CM_CUDA_TRY(cudaMalloc(&t->d6, 48));
    CM_CUDA_TRY(cudaMalloc(&t->dcnt, 16 * nranks));
    cl->tr = std::move(t);
  } else if (transport == CM_TRANSPORT_IN_PROCESS) {
    auto t = std::make_unique<LocalTransport>();
    t->P = nranks, t->rank = rank;
    const std::string key(static_cast<const char*>(id), CM_CLUSTER_ID_BYTES);
    std::lock_guard<std::mutex> lk(g_groups_mu);
    auto& w = g_groups[key];
    t->grp = w.lock();
    if (!t->grp) {
      t->grp = std::make_shared<LocalGroup>(nranks);
      w = t->grp;
    } else if (t->grp->P != nranks) {
      set_error("in-process group joined with a different nranks");
      return CM_INVALID_ARGUMENT;
    }
    cl->tr = std::move(t);
  } else {
    set_error("unknown transport (CM_TRANSPORT_NCCL = 0, CM_TRANSPORT_IN_PROCESS = 1)");
    return CM_INVALID_ARGUMENT;
  }
  *out = cl.release();
  return CM_OK;
}

cm_status cm_cluster_free(cm_cluster* cl) {
  if (!cl) return CM_OK;
  DevGuard dg(cl->device);
  delete cl;
  return CM_OK;
}

cm_status cm_build_slab(cm_cluster* cl, const double* xyz, const uint32_t* gids, uint64_t gid_base,
                        uint64_t n, const cm_build_options* opts, double halo, void* stream,
                        cm_slab** out) {
  if (!cl || !out || (n && !xyz)) {
    set_error("null cluster, points or output");
    return CM_INVALID_ARGUMENT;
  }
  *out = nullptr;
  if (!(halo >= 0.0)) {
    set_error("halo must be >= 0");
    return CM_INVALID_ARGUMENT;
  }
  cm_build_options o;
  if (opts) o = *opts;
  else cm_default_options(&o);
  DevGuard dg(cl->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Transport& T = *cl->tr;
  const int P = T.P;
  auto sl = std::make_unique<cm_slab>();
  sl->cl = cl;
  sl->halo = halo;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const auto h0 = std::chrono::steady_clock::now();
  cudaEventRecord(e0, st);
  std::vector<void*> bufs;
  auto cleanup = [&]() {
    for (void* p : bufs) dev_free(p, st);
    cudaStreamSynchronize(st);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  };
  auto alloc = [&](void** p, size_t bytes) -> bool {
    if (dev_alloc(p, bytes, st) != cudaSuccess) return false;
    bufs.push_back(*p);
    return true;
  };
  cm_status s = CM_OK;
  // 0. inputs on the device
  InBuf in, gin;
  if ((s = stage_input(xyz, n * 24, st, &in)) != CM_OK ||
      (gids && (s = stage_input(gids, n * 4, st, &gin)) != CM_OK)) {
    cleanup();
    return s;
  }
  const double* dx = static_cast<const double*>(in.dev);
  const uint32_t* dg_ids = gids ? static_cast<const uint32_t*>(gin.dev) : nullptr;
  if (!gids && gid_base + n > (1ull << 32)) {
    cleanup();
    set_error("global ids must fit u32");
    return CM_CAPACITY;
  }
  // 1. global bounding box: one MIN all-reduce of (lo, -hi)
  double lo[3], hi[3];
  if ((s = bbox_dev(dx, n, st, lo, hi)) != CM_OK) {
    cleanup();
    return s;
  }
  double v6[6] = {lo[0], lo[1], lo[2], -hi[0], -hi[1], -hi[2]};
  if ((s = T.allreduce_min6(v6, st)) != CM_OK) {
    cleanup();
    return s;
  }
  for (int a = 0; a < 3; ++a) sl->bounds[a] = v6[a], sl->bounds[3 + a] = -v6[3 + a];
  if (!(sl->bounds[0] <= sl->bounds[3])) {
    cleanup();
    set_error("point cloud is empty on every rank");
    return CM_EMPTY_CLOUD;
  }
  // 2. slab edges over the global x extent
  SlabEdges E{};
  E.P = P;
  E.halo = halo;
  const double x0 = sl->bounds[0], x1 = sl->bounds[3];
  for (int p = 0; p < P; ++p) E.e[p] = x0 + (x1 - x0) * (double)p / (double)P;
  E.e[P] = x1;
  sl->edges.assign(E.e, E.e + P + 1);
  if (P > 1 && halo > (x1 - x0) / (double)P) {
    cleanup();
    set_error("halo wider than a slab (would need points from beyond the neighbour slab)");
    return CM_INVALID_ARGUMENT;
  }
  // 3. classify + pack by destination
  unsigned long long* dcount = nullptr;
  if (!alloc(reinterpret_cast<void**>(&dcount), 8 * (2 * P + 1))) {
    cleanup();
    set_error("device allocation failed");
    return CM_CUDA;
  }
  CM_CUDA_TRY(cudaMemsetAsync(dcount, 0, 8 * (2 * P + 1), st));
  if (n) {
    slab_count_kernel<<<grid_of(n), 256, 0, st>>>(dx, n, E, dcount); ::cmg::note_launch();
  }
  std::vector<uint64_t> send_cnt(P), recv_cnt(P), soff(P + 1, 0), roff(P + 1, 0);
  CM_CUDA_TRY(cudaMemcpyAsync(send_cnt.data(), dcount, 8 * P, cudaMemcpyDeviceToHost, st));
  CM_CUDA_TRY(cudaStreamSynchronize(st));
  for (int p = 0; p < P; ++p) soff[p + 1] = soff[p] + send_cnt[p];
  PointRec* sendbuf = nullptr;
  if (!alloc(reinterpret_cast<void**>(&sendbuf), sizeof(PointRec) * std::max<uint64_t>(1, soff[P]))) {
    cleanup();
    set_error("device allocation failed (send buffer)");
    return CM_CUDA;
  }
  {
    std::vector<unsigned long long> cur(soff.begin(), soff.end() - 1);
    CM_CUDA_TRY(cudaMemcpyAsync(dcount + P, cur.data(), 8 * P, cudaMemcpyHostToDevice, st));
    if (n) {
      slab_pack_kernel<<<grid_of(n), 256, 0, st>>>(dx, dg_ids, gid_base, n, E, dcount + P, sendbuf,
                                                   soff[P]);
      ::cmg::note_launch();
    }
    CM_CUDA_TRY(cudaGetLastError());
    CM_CUDA_TRY(cudaStreamSynchronize(st));  // `cur` leaves scope
  }
  // 4. sizes, then the grouped exchange
  if ((s = T.alltoall_u64(send_cnt.data(), recv_cnt.data(), st)) != CM_OK) {
    cleanup();
    return s;
  }
  for (int p = 0; p < P; ++p) roff[p + 1] = roff[p] + recv_cnt[p];
  const uint64_t nl = roff[P];
  if (nl >= (1ull << 32)) {
    cleanup();
    set_error("slab holds 2^32 points or more");
    return CM_CAPACITY;
  }
  PointRec* recvbuf = nullptr;
  if (!alloc(reinterpret_cast<void**>(&recvbuf), sizeof(PointRec) * std::max<uint64_t>(1, nl))) {
    cleanup();
    set_error("device allocation failed (receive buffer)");
    return CM_CUDA;
  }
  {
    std::vector<const void*> sp(P);
    std::vector<void*> rp(P);
    std::vector<uint64_t> sb(P), rb(P);
    for (int p = 0; p < P; ++p) {
      sp[p] = sendbuf + soff[p];
      sb[p] = send_cnt[p] * sizeof(PointRec);
      rp[p] = recvbuf + roff[p];
      rb[p] = recv_cnt[p] * sizeof(PointRec);
    }
    if ((s = T.exchange(sp.data(), sb.data(), rp.data(), rb.data(), st)) != CM_OK) {
      cleanup();
      return s;
    }
  }
  // 5. local records in global-id order
  sl->n_local = nl;
  double* lxyz = nullptr;
  uint32_t* owned = nullptr;
  uint32_t* opos = nullptr;
  if (nl) {
    uint32_t *keys = nullptr, *order = nullptr;
    void* scratch = nullptr;
    if (!alloc(reinterpret_cast<void**>(&keys), 4 * nl) || !alloc(reinterpret_cast<void**>(&order), 4 * nl) ||
        !alloc(&scratch, radix_scratch_bytes<uint32_t>(nl)) ||
        !alloc(reinterpret_cast<void**>(&lxyz), 24 * nl) ||
        !alloc(reinterpret_cast<void**>(&owned), 4 * (nl + 1)) ||
        !alloc(reinterpret_cast<void**>(&opos), 4 * (nl + 1)) ||
        dev_alloc_t(&sl->local_gid, nl, st) != cudaSuccess) {
      cleanup();
      set_error("device allocation failed (local cloud)");
      return CM_CUDA;
    }
    slab_keys_kernel<<<grid_of(nl), 256, 0, st>>>(recvbuf, nl, keys, order); ::cmg::note_launch();
    radix_sort_pairs<uint32_t>(keys, order, nl, 32, scratch, st);
    slab_unpack_kernel<<<grid_of(nl), 256, 0, st>>>(recvbuf, order, nl, lxyz, sl->local_gid, owned);
    ::cmg::note_launch();
    // owned positions: exclusive scan of the flags (total at [nl])
    uint32_t* part = nullptr;
    if (!alloc(reinterpret_cast<void**>(&part), 4 * scan_part_elems(nl))) {
      cleanup();
      set_error("device allocation failed (scan)");
      return CM_CUDA;
    }
    exclusive_scan<uint32_t, uint32_t>(owned, nl, opos, part, 1, st);
    uint32_t n_own = 0;
    CM_CUDA_TRY(cudaMemcpyAsync(&n_own, opos + nl, 4, cudaMemcpyDeviceToHost, st));
    CM_CUDA_TRY(cudaStreamSynchronize(st));
    sl->n_owned = n_own;
    sl->n_halo = nl - n_own;
    if (n_own) {
      if (dev_alloc_t(&sl->owned_xyz, 3 * (uint64_t)n_own, st) != cudaSuccess ||
          dev_alloc_t(&sl->owned_gid, n_own, st) != cudaSuccess) {
        cleanup();
        set_error("device allocation failed (owned centres)");
        return CM_CUDA;
      }
      slab_owned_kernel<<<grid_of(nl), 256, 0, st>>>(lxyz, sl->local_gid, owned, opos, nl,
                                                      sl->owned_xyz, sl->owned_gid);
      ::cmg::note_launch();
    }
    CM_CUDA_TRY(cudaGetLastError());
    // 6. the local index on the global grid
    sl->ix = new cm_index();
    sl->ix->device = cl->device;
    s = build_index(lxyz, nl, o, st, sl->ix, sl->bounds);
    if (s != CM_OK) {
      cleanup();
      cm_free(sl->ix);
      sl->ix = nullptr;
      cm_slab_free(sl.release());
      return s;
    }
    relabel_kernel<<<grid_of(nl), 256, 0, st>>>(sl->ix->rec, sl->ix->ids, nl, sl->local_gid); ::cmg::note_launch();
    CM_CUDA_TRY(cudaGetLastError());
    sl->ix->global_ids = true;
  }
  cudaEventRecord(e1, st);
  CM_CUDA_TRY(cudaStreamSynchronize(st));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  sl->timing.total_ms = ms;
  sl->timing.wall_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count();
  sl->timing.index_ms = sl->ix ? sl->ix->timing.total_ms : 0.0;
  sl->timing.sent_points = soff[P];
  sl->timing.received_points = nl;
  cleanup();
  *out = sl.release();
  return CM_OK;
}

cm_status cm_slab_free(cm_slab* sl) {
  if (!sl) return CM_OK;
  DevGuard dg(sl->cl ? sl->cl->device : 0);
  cudaDeviceSynchronize();
  if (sl->ix) cm_free(sl->ix);
  for (void* p : {(void*)sl->local_gid, (void*)sl->owned_xyz, (void*)sl->owned_gid})
    if (p) cudaFreeAsync(p, 0);
  cudaStreamSynchronize(0);
  delete sl;
  return CM_OK;
}

cm_status cm_slab_info(const cm_slab* sl, cm_slab_info_t* o, double* edges, uint64_t edges_cap) {
  if (!sl || !o) {
    set_error("null slab or output");
    return CM_INVALID_ARGUMENT;
  }
  o->nranks = sl->cl->tr->P;
  o->rank = sl->cl->tr->rank;
  o->n_local = sl->n_local;
  o->n_owned = sl->n_owned;
  o->n_halo = sl->n_halo;
  o->halo = sl->halo;
  for (int a = 0; a < 6; ++a) o->bounds[a] = sl->bounds[a];
  o->timing = sl->timing;
  for (uint64_t i = 0; edges && i < sl->edges.size() && i < edges_cap; ++i) edges[i] = sl->edges[i];
  return CM_OK;
}

const cm_index* cm_slab_index(const cm_slab* sl) { return sl ? sl->ix : nullptr; }

cm_status cm_slab_ids(const cm_slab* sl, uint32_t* owned_gids, uint32_t* local_gids, void* stream) {
  if (!sl) {
    set_error("null slab");
    return CM_INVALID_ARGUMENT;
  }
  DevGuard dg(sl->cl->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (owned_gids && sl->n_owned)
    CM_CUDA_TRY(cudaMemcpyAsync(owned_gids, sl->owned_gid, 4 * sl->n_owned, cudaMemcpyDefault, st));
  if (local_gids && sl->n_local)
    CM_CUDA_TRY(cudaMemcpyAsync(local_gids, sl->local_gid, 4 * sl->n_local, cudaMemcpyDefault, st));
  CM_CUDA_TRY(cudaStreamSynchronize(st));
  return CM_OK;
}

static cm_status slab_centres(const cm_slab* sl, double r, const double** q, uint64_t* nq) {
  if (!sl) {
    set_error("null slab");
    return CM_INVALID_ARGUMENT;
  }
  if (r > sl->halo && sl->cl->tr->P > 1) {
    set_error("radius exceeds the slab halo: neighbour sets would be incomplete");
    return CM_INVALID_ARGUMENT;
  }
  if (!*q) {
    *q = sl->owned_xyz;
    *nq = sl->n_owned;
  }
  if (!sl->ix) {
    set_error("slab holds no points");
    return CM_EMPTY_CLOUD;
  }
  return CM_OK;
}

// Radius search for centres inside this rank's slab (q = NULL: every owned
// point, in ascending global-id order); columns are global ids, rows sorted.
cm_status cm_slab_radius_search(const cm_slab* sl, const double* q, uint64_t nq, int kernel,
                                double r, void* stream, cm_csr** out) {
  cm_status s = slab_centres(sl, r, &q, &nq);
  if (s != CM_OK) return s;
  return cm_radius_search(sl->ix, q, nq, kernel, r, stream, out);
}

// cm_radius_digest over global ids for centres in this slab (q = NULL: owned).
cm_status cm_slab_radius_digest(const cm_slab* sl, const double* q, uint64_t nq, int kernel,
                                double r, uint32_t* counts, uint64_t* digests, void* stream) {
  cm_status s = slab_centres(sl, r, &q, &nq);
  if (s != CM_OK) return s;
  return cm_radius_digest(sl->ix, q, nq, kernel, r, counts, digests, stream);
}

}  // extern "C"
