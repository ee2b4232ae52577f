// LAS ingestion on sm_100a — replaces read_las (io.cpp:33-106).
//
// The header (a few hundred bytes) is checked on the host with the
// reference's checks, messages and order (io.cpp:38-89); the point records
// are decoded on the device: coordinate = raw * scale + offset with the
// reference's exact fp64 arithmetic (int32 -> double, __dmul_rn, __dadd_rn:
// no FMA), io.cpp:97-103.
//
// Decode kernel: HBM-bound byte work (record_length bytes in, 24 bytes out
// per point). A block takes a tile of T consecutive records, stages the
// tile's bytes in shared memory with 16-byte vector loads (any source
// alignment; byte loads only at the buffer's ragged end), then each thread
// extracts its record's X, Y, Z from shared memory (four aligned words and a
// funnel shift) and writes its 24-byte point (the block's output is one
// contiguous, coalesced stretch).
#include <cstdio>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "index.cuh"

#define LAS_TRY(expr)              \
  do {                             \
    const cm_status _s = (expr);   \
    if (_s != CM_OK) return _s;    \
  } while (0)

namespace cmg {

int sm_count();

namespace {

constexpr uint32_t kLasHeader12 = 227;  // io.cpp:30

template <class T>
T rd(const unsigned char* b, size_t off) {
  T v;
  std::memcpy(&v, b + off, sizeof(T));
  return v;  // little-endian host, as the reference assumes (io.cpp:17-21)
}

// io.cpp:38-89, in order. `name` only feeds the messages.
cm_status parse_header(const unsigned char* b, uint64_t n, const std::string& name,
                       cm_las_header* h) {
  if (n < kLasHeader12 || std::memcmp(b, "LASF", 4) != 0) {
    set_error("bad LAS magic at byte 0 in " + name);
    return CM_PARSE;
  }
  std::memset(h, 0, sizeof(*h));
  h->version_major = b[24];
  h->version_minor = b[25];
  if (h->version_major != 1 || h->version_minor < 2 || h->version_minor > 4) {
    set_error("unsupported LAS version " + std::to_string(h->version_major) + "." +
              std::to_string(h->version_minor));
    return CM_PARSE;
  }
  h->header_size = rd<uint16_t>(b, 94);
  h->data_offset = rd<uint32_t>(b, 96);
  h->point_format = b[104];
  if (h->point_format > 8) {
    set_error("unsupported LAS point record format " + std::to_string(h->point_format));
    return CM_PARSE;
  }
  h->record_length = rd<uint16_t>(b, 105);
  if (h->record_length < 12) {
    set_error("LAS point record length " + std::to_string(h->record_length) + " is too short");
    return CM_PARSE;
  }
  h->point_count = rd<uint32_t>(b, 107);
  if (h->point_count == 0 && h->version_minor == 4 && h->header_size >= 255) {
    // the 64-bit count of LAS 1.4 (io.cpp:63-65); bytes past the image read as 0
    unsigned char c8[8] = {};
    for (int i = 0; i < 8; ++i)
      if (247 + i < n) c8[i] = b[247 + i];
    std::memcpy(&h->point_count, c8, 8);
  }
  for (int a = 0; a < 3; ++a) h->scale[a] = rd<double>(b, 131 + 8 * a);
  if (!(h->scale[0] > 0.0) || !(h->scale[1] > 0.0) || !(h->scale[2] > 0.0)) {
    set_error("non-positive LAS scale factor at byte 131");
    return CM_PARSE;
  }
  for (int a = 0; a < 3; ++a) h->offset[a] = rd<double>(b, 155 + 8 * a);
  for (int a = 0; a < 3; ++a) {  // max then min per axis (io.cpp:75-80)
    h->bounds_max[a] = rd<double>(b, 179 + 16 * a);
    h->bounds_min[a] = rd<double>(b, 187 + 16 * a);
  }
  if (h->data_offset < h->header_size || h->data_offset > n) {
    set_error("LAS point data offset " + std::to_string(h->data_offset) + " is out of range");
    return CM_PARSE;
  }
  return CM_OK;
}

// The reference stops at the first record that does not fit (io.cpp:92-96).
cm_status check_records(const cm_las_header& h, uint64_t n) {
  const uint64_t avail = (n - h.data_offset) / h.record_length;
  if (avail < h.point_count) {
    set_error("truncated LAS point record " + std::to_string(avail) + " at byte " +
              std::to_string(h.data_offset + avail * h.record_length));
    return CM_PARSE;
  }
  return CM_OK;
}

struct LasScale {
  double sx, sy, sz, ox, oy, oz;
};

__device__ __forceinline__ void las_point(int32_t rx, int32_t ry, int32_t rz, const LasScale& s,
                                          double* out) {
  out[0] = __dadd_rn(__dmul_rn((double)rx, s.sx), s.ox);
  out[1] = __dadd_rn(__dmul_rn((double)ry, s.sy), s.oy);
  out[2] = __dadd_rn(__dmul_rn((double)rz, s.sz), s.oz);
}

// Tiles of T records staged through shared memory. `recs` points at record 0
// (any alignment); `end` bounds every read.
__global__ void __launch_bounds__(256) las_decode_kernel(const unsigned char* __restrict__ recs,
                                                         uint64_t n, uint32_t rl, uint32_t T,
                                                         const unsigned char* end, LasScale s,
                                                         double* __restrict__ out) {
  extern __shared__ __align__(16) uint32_t lsm[];
  const uint64_t ntiles = (n + T - 1) / T;
  for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const uint64_t r0 = tile * T;
    const uint32_t cnt = (uint32_t)(n - r0 < T ? n - r0 : T);
    const unsigned char* a = recs + r0 * rl;
    const unsigned char* as = reinterpret_cast<const unsigned char*>(
        reinterpret_cast<uintptr_t>(a) & ~(uintptr_t)15);
    const uint32_t lead = (uint32_t)(a - as);
    const uint32_t bytes = lead + cnt * rl;
    const uint32_t nvec = (bytes + 15) / 16;
    for (uint32_t v = threadIdx.x; v < nvec; v += blockDim.x) {
      const unsigned char* src = as + 16 * (size_t)v;
      uint4 w;
      if (src + 16 <= end) {
        w = __ldg(reinterpret_cast<const uint4*>(src));
      } else {  // the image's ragged end: bytes that exist, zeros past it
        unsigned char t[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) t[k] = src + k < end ? src[k] : 0;
        std::memcpy(&w, t, 16);
      }
      reinterpret_cast<uint4*>(lsm)[v] = w;
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < cnt; i += blockDim.x) {
      const uint32_t o = lead + i * rl;
      const uint32_t q = o >> 2, sh = (o & 3) * 8;
      const uint32_t w0 = lsm[q], w1 = lsm[q + 1], w2 = lsm[q + 2], w3 = lsm[q + 3];
      const int32_t rx = (int32_t)__funnelshift_r(w0, w1, sh);
      const int32_t ry = (int32_t)__funnelshift_r(w1, w2, sh);
      const int32_t rz = (int32_t)__funnelshift_r(w2, w3, sh);
      las_point(rx, ry, rz, s, out + 3 * (r0 + i));
    }
    __syncthreads();
  }
}

// Records too long to stage a useful tile (record_length > 1536): byte loads.
__global__ void las_decode_direct_kernel(const unsigned char* __restrict__ recs, uint64_t n,
                                         uint32_t rl, LasScale s, double* __restrict__ out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned char* p = recs + i * rl;
    int32_t v[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const uint32_t u = (uint32_t)p[4 * a] | ((uint32_t)p[4 * a + 1] << 8) |
                         ((uint32_t)p[4 * a + 2] << 16) | ((uint32_t)p[4 * a + 3] << 24);
      v[a] = (int32_t)u;
    }
    las_point(v[0], v[1], v[2], s, out + 3 * i);
  }
}

cm_status launch_decode(const unsigned char* recs, uint64_t n, uint32_t rl,
                        const unsigned char* end, const cm_las_header& h, double* out,
                        cudaStream_t st) {
  if (n == 0) return CM_OK;
  const LasScale s{h.scale[0], h.scale[1], h.scale[2], h.offset[0], h.offset[1], h.offset[2]};
  if (rl > 1536) {
    const unsigned grid = (unsigned)std::min<uint64_t>((n + 255) / 256, (uint64_t)sm_count() * 16);
    las_decode_direct_kernel<<<grid, 256, 0, st>>>(recs, n, rl, s, out); note_launch();
    CM_CUDA_TRY(cudaGetLastError());
    return CM_OK;
  }
  // T records per tile: as many as 48 KB of staging allows, up to 256
  uint32_t T = 256;
  while (T > 32 && (size_t)T * rl + 32 > 48 * 1024) T -= 32;
  const size_t smem = ((size_t)T * rl + 16 + 15) / 16 * 16 + 16;
  const uint64_t tiles = (n + T - 1) / T;
  const unsigned grid = (unsigned)std::min<uint64_t>(tiles, (uint64_t)sm_count() * 8);
  las_decode_kernel<<<grid, 256, smem, st>>>(recs, n, rl, T, end, s, out); note_launch();
  CM_CUDA_TRY(cudaGetLastError());
  return CM_OK;
}

// Header bytes of an image that may live in device memory.
cm_status fetch_header(const void* bytes, uint64_t nbytes, std::vector<unsigned char>* hb) {
  const uint64_t take = std::min<uint64_t>(nbytes, 375);  // the largest (1.4) header
  hb->assign(take, 0);
  if (!take) return CM_OK;
  if (is_device_ptr(bytes))
    CM_CUDA_TRY(cudaMemcpy(hb->data(), bytes, take, cudaMemcpyDeviceToHost));
  else
    std::memcpy(hb->data(), bytes, take);
  return CM_OK;
}

cm_status decode_image(const void* bytes, uint64_t nbytes, const std::string& name,
                       double* xyz, uint64_t cap, cm_las_header* hdr, int device,
                       cudaStream_t st) {
  std::vector<unsigned char> hb;
  LAS_TRY(fetch_header(bytes, nbytes, &hb));
  hb.resize(375, 0);  // header fields only; ranges are checked against nbytes
  cm_las_header h;
  LAS_TRY(parse_header(hb.data(), nbytes, name, &h));
  LAS_TRY(check_records(h, nbytes));
  if (hdr) *hdr = h;
  if (!xyz) return CM_OK;
  if (cap < h.point_count) {
    set_error("xyz capacity " + std::to_string(cap) + " < LAS point count " +
              std::to_string(h.point_count));
    return CM_INVALID_ARGUMENT;
  }
  const uint64_t n = h.point_count;
  if (n == 0) return CM_OK;
  const uint64_t rbytes = n * h.record_length;
  const unsigned char* recs = nullptr;
  unsigned char* owned_in = nullptr;
  if (is_device_ptr(bytes)) {
    recs = static_cast<const unsigned char*>(bytes) + h.data_offset;
  } else {
    CM_CUDA_TRY(dev_alloc(reinterpret_cast<void**>(&owned_in), rbytes + 16, st));
    const cudaError_t e = cudaMemcpyAsync(owned_in, static_cast<const unsigned char*>(bytes) + h.data_offset,
                                          rbytes, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) {
      dev_free(owned_in, st);
      set_error(std::string("cudaMemcpyAsync: ") + cudaGetErrorString(e));
      return CM_CUDA;
    }
    recs = owned_in;
  }
  double* out = xyz;
  double* owned_out = nullptr;
  const bool host_out = !is_device_ptr(xyz);
  cm_status s = CM_OK;
  if (host_out) {
    if (dev_alloc(reinterpret_cast<void**>(&owned_out), n * 24, st) != cudaSuccess) {
      set_error("device allocation failed (LAS points)");
      s = CM_CUDA;
    }
    out = owned_out;
  }
  if (s == CM_OK) s = launch_decode(recs, n, h.record_length, recs + rbytes, h, out, st);
  if (s == CM_OK && host_out) {
    if (cudaMemcpyAsync(xyz, owned_out, n * 24, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess) {
      set_error("LAS point copy-back failed");
      s = CM_CUDA;
    }
  }
  if (owned_in) dev_free(owned_in, st);
  if (owned_out) dev_free(owned_out, st);
  if (host_out || owned_in) cudaStreamSynchronize(st);
  (void)device;
  return s;
}

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
}  // namespace cmg

extern "C" {

cm_status cm_las_parse_header(const void* bytes, uint64_t nbytes, cm_las_header* out) {
  if (!out || (nbytes && !bytes)) {
    cmg::set_error("null LAS image or header pointer");
    return CM_INVALID_ARGUMENT;
  }
  std::vector<unsigned char> hb(375, 0);  // header fields only (host memory)
  if (nbytes) std::memcpy(hb.data(), bytes, std::min<uint64_t>(nbytes, 375));
  return cmg::parse_header(hb.data(), nbytes, "<memory>", out);
}

cm_status cm_las_decode(const void* bytes, uint64_t nbytes, double* xyz, uint64_t xyz_capacity,
                        cm_las_header* hdr, int device, void* stream) {
  if (nbytes && !bytes) {
    cmg::set_error("null LAS image");
    return CM_INVALID_ARGUMENT;
  }
  cmg::DevGuard dg(device);
  return cmg::decode_image(bytes, nbytes, "<memory>", xyz, xyz_capacity, hdr, device,
                           static_cast<cudaStream_t>(stream));
}

cm_status cm_las_read(const char* path, double* xyz, uint64_t xyz_capacity, cm_las_header* hdr,
                      int device, void* stream) {
  if (!path) {
    cmg::set_error("null path");
    return CM_INVALID_ARGUMENT;
  }
  std::ifstream in(path, std::ios::binary);
  if (!in) {
    cmg::set_error(std::string("cannot open ") + path);
    return CM_IO;
  }
  std::vector<char> buf((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  cmg::DevGuard dg(device);
  return cmg::decode_image(buf.data(), buf.size(), path, xyz, xyz_capacity, hdr, device,
                           static_cast<cudaStream_t>(stream));
}

}  // extern "C"
