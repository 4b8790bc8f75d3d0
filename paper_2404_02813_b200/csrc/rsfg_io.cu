// rsfg_io.cu -- volume I/O straight to the device and overlap metrics
// (reference volume_io.cpp:24-137, validation.cpp:13-52).
//
//  * read: the .vmh header is parsed on the host with the reference's rules
//    and messages; the payload streams through two pinned staging buffers in
//    chunks -- disk read of chunk k+1 overlaps the H2D copy of chunk k -- and
//    moves across PCIe in its stored width (1 or 2 bytes per voxel for u8 /
//    u16), the conversion to f32 (u16 rescaled onto [0, 255] with the
//    reference's f32 scale) running on the device;
//  * dice / jaccard: foreground = value > 0.5, exact 64-bit counts.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/rsfg.h"
#include "rsfg_internal.h"

namespace {

int ioerr(const std::string& m) {
  rsfg::set_error(m);
  return RSFG_ERR_IO;
}

std::string trim(const std::string& s) {
  const auto a = s.find_first_not_of(" \t\r\n");
  if (a == std::string::npos) return "";
  const auto b = s.find_last_not_of(" \t\r\n");
  return s.substr(a, b - a + 1);
}

struct Header {
  int nx = 0, ny = 0, nz = 0;
  double sx = 1, sy = 1, sz = 1;
  std::string dtype, data;
  bool has_range = false;
  float lo = 0, hi = 0;
  size_t elem = 4;
  std::string raw_path;
};

// read_volume's header rules and messages (volume_io.cpp:24-76).
int parse_header(const char* path, Header& h) {
  const std::string hp = path ? path : "";
  std::ifstream in(hp);
  if (!in) return ioerr("cannot open volume header: " + hp);
  bool have_dims = false, have_dtype = false, have_data = false;
  std::string line;
  while (std::getline(in, line)) {
    line = trim(line);
    if (line.empty() || line[0] == '#') continue;
    const auto colon = line.find(':');
    if (colon == std::string::npos) return ioerr("garbled header line in " + hp + ": " + line);
    const std::string key = trim(line.substr(0, colon)), val = trim(line.substr(colon + 1));
    std::istringstream vs(val);
    if (key == "dims") {
      if (!(vs >> h.nx >> h.ny >> h.nz) || h.nx <= 0 || h.ny <= 0 || h.nz <= 0)
        return ioerr("bad dims in " + hp + ": " + val);
      have_dims = true;
    } else if (key == "spacing") {
      if (!(vs >> h.sx >> h.sy >> h.sz)) return ioerr("bad spacing in " + hp + ": " + val);
    } else if (key == "dtype") {
      h.dtype = val;
      have_dtype = true;
    } else if (key == "data") {
      h.data = val;
      have_data = true;
    } else if (key == "range") {
      if (!(vs >> h.lo >> h.hi)) return ioerr("bad range in " + hp + ": " + val);
      h.has_range = true;
    } else {
      return ioerr("unknown header key '" + key + "' in " + hp);
    }
  }
  if (!have_dims || !have_dtype || !have_data) return ioerr("header missing dims/dtype/data: " + hp);
  if (h.dtype == "u8") h.elem = 1;
  else if (h.dtype == "u16") h.elem = 2;
  else if (h.dtype == "f32") h.elem = 4;
  else return ioerr("unsupported dtype '" + h.dtype + "' in " + hp);
  const auto slash = hp.find_last_of('/');
  h.raw_path = (slash == std::string::npos ? std::string() : hp.substr(0, slash + 1)) + h.data;
  return RSFG_OK;
}

// u8 -> f32, u16 (little-endian) -> f32 * 255/65535, f32 copied.
__global__ void convert_kernel(const unsigned char* __restrict__ src, float* __restrict__ dst, size_t n, int elem) {
  constexpr float scale = 255.0f / 65535.0f;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    if (elem == 1) {
      dst[i] = (float)src[i];
    } else if (elem == 2) {
      const unsigned lo = src[2 * i], hi = src[2 * i + 1];
      dst[i] = (float)(lo | (hi << 8)) * scale;
    } else {
      float v;
      memcpy(&v, src + 4 * i, 4);
      dst[i] = v;
    }
  }
}

__global__ void overlap_kernel(const float* __restrict__ a, const float* __restrict__ b, size_t n,
                               unsigned long long* __restrict__ cnt) {
  unsigned long long ca = 0, cb = 0, cab = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const bool fa = a[i] > 0.5f, fb = b[i] > 0.5f;
    ca += fa;
    cb += fb;
    cab += fa && fb;
  }
  for (int o = 16; o; o >>= 1) {
    ca += __shfl_down_sync(0xffffffffu, ca, o);
    cb += __shfl_down_sync(0xffffffffu, cb, o);
    cab += __shfl_down_sync(0xffffffffu, cab, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(cnt, ca);
    atomicAdd(cnt + 1, cb);
    atomicAdd(cnt + 2, cab);
  }
}

}  // namespace

extern "C" {

__attribute__((visibility("default"))) int rsfg_volume_info(const char* header, int32_t* nx, int32_t* ny,
                                                            int32_t* nz, double* spacing3, int32_t* elem_bytes) {
  Header h;
  if (int rc = parse_header(header, h)) return rc;
  if (nx) *nx = h.nx;
  if (ny) *ny = h.ny;
  if (nz) *nz = h.nz;
  if (spacing3) spacing3[0] = h.sx, spacing3[1] = h.sy, spacing3[2] = h.sz;
  if (elem_bytes) *elem_bytes = (int32_t)h.elem;
  return RSFG_OK;
}

__attribute__((visibility("default"))) int rsfg_read_volume_device(const char* header, float* d_out, int64_t capacity,
                                                                   int32_t device, float* range2,
                                                                   int64_t* h2d_bytes) {
  Header h;
  if (int rc = parse_header(header, h)) return rc;
  const size_t n = (size_t)h.nx * h.ny * h.nz;
  if (!d_out || capacity < (int64_t)n) {
    rsfg::set_error("read_volume: output buffer smaller than the volume");
    return RSFG_ERR_SHAPE;
  }
  std::ifstream raw(h.raw_path, std::ios::binary);
  if (!raw) return ioerr("cannot open payload: " + h.raw_path);
  raw.seekg(0, std::ios::end);
  const size_t bytes = (size_t)raw.tellg();
  raw.seekg(0);
  const size_t expected = n * h.elem;
  if (bytes != expected)
    return ioerr("payload size mismatch for " + std::string(header) + ": header implies " + std::to_string(expected) +
                 " bytes, file has " + std::to_string(bytes));
  if (cudaSetDevice(device) != cudaSuccess) {
    rsfg::set_error("read_volume: bad device");
    return RSFG_ERR_CUDA;
  }
  const size_t chunk_vox = (size_t)1 << 24;  // 16 Mi voxels per chunk
  const size_t chunk = chunk_vox * h.elem;
  unsigned char* pin[2] = {nullptr, nullptr};
  unsigned char* dev[2] = {nullptr, nullptr};
  cudaStream_t st;
  cudaEvent_t done[2];
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaEventCreateWithFlags(&done[0], cudaEventDisableTiming);
  cudaEventCreateWithFlags(&done[1], cudaEventDisableTiming);
  int rc = RSFG_OK;
  if (cudaMallocHost(&pin[0], chunk) != cudaSuccess || cudaMallocHost(&pin[1], chunk) != cudaSuccess ||
      (h.elem != 4 && (cudaMalloc(&dev[0], chunk) != cudaSuccess || cudaMalloc(&dev[1], chunk) != cudaSuccess))) {
    rsfg::set_error("read_volume: out of memory for staging buffers");
    rc = RSFG_ERR_OOM;
  }
  size_t moved = 0;
  for (size_t off = 0, k = 0; rc == RSFG_OK && off < n; off += chunk_vox, ++k) {
    const int b = (int)(k & 1);
    const size_t nv = std::min(chunk_vox, n - off), nb = nv * h.elem;
    cudaEventSynchronize(done[b]);  // staging buffer b free again (chunk k-2 done)
    raw.read(reinterpret_cast<char*>(pin[b]), (std::streamsize)nb);
    if (!raw) {
      rc = ioerr("short read from payload: " + h.raw_path);
      break;
    }
    if (h.elem == 4) {
      cudaMemcpyAsync(d_out + off, pin[b], nb, cudaMemcpyHostToDevice, st);
    } else {
      cudaMemcpyAsync(dev[b], pin[b], nb, cudaMemcpyHostToDevice, st);
      convert_kernel<<<148 * 4, 256, 0, st>>>(dev[b], d_out + off, nv, (int)h.elem);
    }
    cudaEventRecord(done[b], st);
    moved += nb;
  }
  if (cudaStreamSynchronize(st) != cudaSuccess && rc == RSFG_OK) {
    rsfg::set_error("read_volume: CUDA error");
    rc = RSFG_ERR_CUDA;
  }
  if (rc == RSFG_OK && range2) {
    if (h.has_range) {
      range2[0] = h.lo, range2[1] = h.hi;
    } else {  // value_range = min_max() (volume_io.cpp:111)
      unsigned int* mm = nullptr;
      const unsigned int init[2] = {0xffffffffu, 0u};
      cudaMalloc(&mm, 2 * sizeof(unsigned int));
      cudaMemcpyAsync(mm, init, sizeof init, cudaMemcpyHostToDevice, st);
      rsfg::Geom g{h.nx, h.ny, h.nz, 0, h.nz, (long long)h.nx * h.ny};
      rsfg::launch_minmax(g, d_out, 0, h.nz, mm, st);
      unsigned int out[2];
      cudaMemcpyAsync(out, mm, sizeof out, cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      cudaFree(mm);
      range2[0] = rsfg::decode_ordered(out[0]);
      range2[1] = rsfg::decode_ordered(out[1]);
    }
  }
  if (h2d_bytes) *h2d_bytes = (int64_t)moved;
  cudaFreeHost(pin[0]);
  cudaFreeHost(pin[1]);
  cudaFree(dev[0]);
  cudaFree(dev[1]);
  cudaEventDestroy(done[0]);
  cudaEventDestroy(done[1]);
  cudaStreamDestroy(st);
  return rc;
}

// write_volume (volume_io.cpp:115-137) from a DEVICE field: f32 payload next
// to the header, range = min_max unless range2 is given.
__attribute__((visibility("default"))) int rsfg_write_volume_device(const char* header, const float* d_v, int32_t nx,
                                                                    int32_t ny, int32_t nz, const double* spacing3,
                                                                    const float* range2, int32_t device) {
  if (!header || !d_v || nx <= 0 || ny <= 0 || nz <= 0) {
    rsfg::set_error("write_volume: data length does not match dims");
    return RSFG_ERR_SHAPE;
  }
  const size_t n = (size_t)nx * ny * nz;
  std::vector<float> host(n);
  if (cudaSetDevice(device) != cudaSuccess || cudaMemcpy(host.data(), d_v, n * 4, cudaMemcpyDeviceToHost) != cudaSuccess) {
    rsfg::set_error("write_volume: CUDA error");
    return RSFG_ERR_CUDA;
  }
  std::string hp(header), rp = hp;
  const auto dot = rp.find_last_of('.'), slash = rp.find_last_of('/');
  if (dot != std::string::npos && (slash == std::string::npos || dot > slash)) rp = rp.substr(0, dot);
  rp += ".raw";
  {
    std::ofstream raw(rp, std::ios::binary | std::ios::trunc);
    if (!raw) return ioerr("cannot write payload: " + rp);
    raw.write(reinterpret_cast<const char*>(host.data()), (std::streamsize)(n * 4));
    if (!raw) return ioerr("short write to payload: " + rp);
  }
  float lo, hi;
  if (range2) {
    lo = range2[0], hi = range2[1];
  } else {
    lo = hi = host[0];
    for (float v : host) lo = std::min(lo, v), hi = std::max(hi, v);
  }
  std::ofstream out(hp, std::ios::trunc);
  if (!out) return ioerr("cannot write header: " + hp);
  const double s[3] = {spacing3 ? spacing3[0] : 1.0, spacing3 ? spacing3[1] : 1.0, spacing3 ? spacing3[2] : 1.0};
  const std::string fname = slash == std::string::npos ? rp : rp.substr(rp.find_last_of('/') + 1);
  out << "dims: " << nx << " " << ny << " " << nz << "\n";
  out << "spacing: " << s[0] << " " << s[1] << " " << s[2] << "\n";
  out << "dtype: f32\n";
  out << "data: " << fname << "\n";
  out << "range: " << lo << " " << hi << "\n";
  if (!out) return ioerr("short write to header: " + hp);
  return RSFG_OK;
}

// dice / jaccard (validation.cpp:41-52) of two DEVICE volumes.
__attribute__((visibility("default"))) int rsfg_overlap_device(const float* d_a, const float* d_b, int64_t n,
                                                               int32_t device, double* dice, double* jaccard) {
  if (!d_a || !d_b || n < 0) {
    rsfg::set_error("overlap metric: null buffer");
    return RSFG_ERR_STATE;
  }
  if (cudaSetDevice(device) != cudaSuccess) return RSFG_ERR_CUDA;
  unsigned long long* cnt = nullptr;
  if (cudaMalloc(&cnt, 3 * sizeof(unsigned long long)) != cudaSuccess) return RSFG_ERR_OOM;
  cudaMemset(cnt, 0, 3 * sizeof(unsigned long long));
  overlap_kernel<<<148 * 8, 256>>>(d_a, d_b, (size_t)n, cnt);
  unsigned long long c[3];
  const cudaError_t e = cudaMemcpy(c, cnt, sizeof c, cudaMemcpyDeviceToHost);
  cudaFree(cnt);
  if (e != cudaSuccess) return RSFG_ERR_CUDA;
  if (dice) *dice = (c[0] + c[1] == 0) ? 1.0 : 2.0 * (double)c[2] / (double)(c[0] + c[1]);
  const unsigned long long uni = c[0] + c[1] - c[2];
  if (jaccard) *jaccard = uni == 0 ? 1.0 : (double)c[2] / (double)uni;
  return RSFG_OK;
}

}  // extern "C"
