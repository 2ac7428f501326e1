// Device utilities: the reference's deterministic input generator, pitched
// copies, ring reset, and the launch counter.
#include <atomic>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include "common.cuh"
#include "kernels.h"

namespace pcotgpu {

namespace {

std::atomic<uint64_t> g_launches{0};

// reference exec.cpp:21-28: splitmix64(fnv1a(name) ^ flat*phi) >> 11, * 2^-53
PCOT_DEV double init_value_dev(uint64_t h, uint64_t flat) {
  uint64_t x = h ^ (flat * 0x9E3779B97F4A7C15ULL);
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  x ^= x >> 31;
  return double(x >> 11) * 0x1.0p-53;  // exact: 53-bit integer times a power of two
}

__global__ void fill2d_kernel(double* dst, int64_t ld, int64_t nrows, int64_t ncols, uint64_t h,
                              uint64_t flat0) {
  const int64_t total = nrows * ncols;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = e / ncols, c = e - r * ncols;
    dst[r * ld + c] = init_value_dev(h, flat0 + uint64_t(e));
  }
}

__global__ void fill3d_kernel(Grid3D g, uint64_t h) {
  const int64_t n = g.n, total = n * n * n;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e / (n * n), rem = e - i * n * n, j = rem / n, k = rem - j * n;
    g.origin[i * g.pitch_i + j * g.pitch_j + k] = init_value_dev(h, uint64_t(e));
  }
}

__global__ void copy_rows_kernel(double* dst, int64_t ldd, const double* src, int64_t lds,
                                 int64_t nrows, int64_t ncols, int64_t pd, int64_t rpp) {
  const int64_t total = nrows * ncols;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = e / ncols, c = e - r * ncols;
    const int64_t drow = rpp ? (r / rpp) * pd + (r % rpp) * ldd : r * ldd;
    dst[drow + c] = src[r * lds + c];
  }
}

// Copy that maps the one bit pattern the Gauss-Seidel pipeline reserves as its
// "not yet written" edge-slot sentinel (0xffff...ffff, a NaN) to its neighbour
// NaN 0xffff...fffe.  The device's fp64 arithmetic propagates an input NaN's
// payload (measured: without this an input cell holding the sentinel bits
// stalled the band below), so with no such input no computed value can carry
// it; any other input bit pattern is copied unchanged.
__global__ void copy_rows_nosentinel_kernel(double* dst, int64_t ldd, const double* src, int64_t lds,
                                            int64_t nrows, int64_t ncols) {
  const int64_t total = nrows * ncols;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = e / ncols, c = e - r * ncols;
    long long v = __double_as_longlong(src[r * lds + c]);
    if (v == -1LL) v = -2LL;
    dst[r * ldd + c] = __longlong_as_double(v);
  }
}

__global__ void zero_ring2d_kernel(double* o, int64_t ld, int64_t n) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < 4 * n;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t side = e / n, p = e - side * n;
    int64_t r, c;
    if (side == 0) r = 0, c = p;
    else if (side == 1) r = n - 1, c = p;
    else if (side == 2) r = p, c = 0;
    else r = p, c = n - 1;
    o[r * ld + c] = 0.0;
  }
}

__global__ void zero_ring3d_kernel(Grid3D g) {
  const int64_t n = g.n, total = n * n * n;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e / (n * n), rem = e - i * n * n, j = rem / n, k = rem - j * n;
    if (i == 0 || j == 0 || k == 0 || i == n - 1 || j == n - 1 || k == n - 1)
      g.origin[i * g.pitch_i + j * g.pitch_j + k] = 0.0;
  }
}

int grid_for(int64_t total) {
  int64_t b = (total + 255) / 256;
  if (b > 148 * 32) b = 148 * 32;
  if (b < 1) b = 1;
  return int(b);
}

}  // namespace

uint64_t launches() { return g_launches.load(); }
void count_launch(uint64_t n) { g_launches += n; }

cudaError_t fill_init_value(double* dst, int64_t ld, int64_t nrows, int64_t ncols,
                            uint64_t name_hash, uint64_t flat0, cudaStream_t stream) {
  if (nrows <= 0 || ncols <= 0) return cudaSuccess;
  fill2d_kernel<<<grid_for(nrows * ncols), 256, 0, stream>>>(dst, ld, nrows, ncols, name_hash,
                                                             flat0);
  count_launch();
  return cudaGetLastError();
}

cudaError_t fill_init_value_3d(const Grid3D& g, uint64_t name_hash, cudaStream_t stream) {
  if (g.n <= 0) return cudaSuccess;
  fill3d_kernel<<<grid_for(g.n * g.n * g.n), 256, 0, stream>>>(g, name_hash);
  count_launch();
  return cudaGetLastError();
}

cudaError_t copy_rows(double* dst, int64_t ldd, const double* src, int64_t lds, int64_t nrows,
                      int64_t ncols, cudaStream_t stream, int64_t pd, int64_t rpp) {
  if (nrows <= 0 || ncols <= 0) return cudaSuccess;
  copy_rows_kernel<<<grid_for(nrows * ncols), 256, 0, stream>>>(dst, ldd, src, lds, nrows, ncols,
                                                                pd, rpp);
  count_launch();
  return cudaGetLastError();
}

cudaError_t copy_rows_nosentinel(double* dst, int64_t ldd, const double* src, int64_t lds, int64_t nrows,
                                 int64_t ncols, cudaStream_t stream) {
  if (nrows <= 0 || ncols <= 0) return cudaSuccess;
  copy_rows_nosentinel_kernel<<<grid_for(nrows * ncols), 256, 0, stream>>>(dst, ldd, src, lds, nrows, ncols);
  count_launch();
  return cudaGetLastError();
}

cudaError_t zero_ring_2d(double* origin, int64_t ld, int64_t n, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  zero_ring2d_kernel<<<grid_for(4 * n), 256, 0, stream>>>(origin, ld, n);
  count_launch();
  return cudaGetLastError();
}

cudaError_t zero_ring_3d(const Grid3D& g, cudaStream_t stream) {
  if (g.n <= 0) return cudaSuccess;
  zero_ring3d_kernel<<<grid_for(g.n * g.n * g.n), 256, 0, stream>>>(g);
  count_launch();
  return cudaGetLastError();
}

// One-time per (kernel, device, block, smem) preparation, thread-safe: the
// dynamic shared-memory opt-in is a per-device function attribute, so a
// process driving several devices (or several host threads) must not share a
// single "done" flag.
cudaError_t kernel_slots(const void* fn, int nthreads, size_t smem, int* slots) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  using Key = std::tuple<const void*, int, int, size_t>;
  static std::mutex mu;
  static std::map<Key, int> cache;
  const Key key{fn, dev, nthreads, smem};
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(key);
  if (it != cache.end()) {
    if (slots) *slots = it->second;
    return cudaSuccess;
  }
  if ((e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem))) !=
      cudaSuccess)
    return e;
  int occ = 0, sms = 0;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, nthreads, smem)) != cudaSuccess)
    return e;
  const int s = occ * sms;  // 0 when the kernel cannot be resident at all
  cache[key] = s;
  if (slots) *slots = s;
  return cudaSuccess;
}

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v && *v ? std::atoi(v) : dflt;
}

}  // namespace pcotgpu
