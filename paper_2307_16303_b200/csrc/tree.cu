// Octree build on the device: Morton codes -> stable radix sort -> depth
// selection -> node offsets -> permuted SoA coordinates.
// Mirrors reference proj/src/octree.cpp:76-171 (build_tree) bit for bit.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "common.cuh"
#include "kernels.h"

namespace h3db {

namespace {

// grid_coord (octree.cpp:67-72): trunc((x - lo) * inv_w * cells), clamped.
// __dsub_rn/__dmul_rn keep the exact rounding sequence (no FMA contraction).
__device__ __forceinline__ long long grid_coord(double x, long long cells) {
  const double t = __dmul_rn(__dmul_rn(__dsub_rn(x, -1.0), 0.5), static_cast<double>(cells));
  long long k = __double2ll_rz(t);
  if (k < 0) k = 0;
  if (k >= cells) k = cells - 1;
  return k;
}

// morton_encode (octree.cpp:30-38): bit b of ix/iy/iz -> bits 3b/3b+1/3b+2.
__device__ __forceinline__ unsigned long long morton(long long ix, long long iy, long long iz,
                                                     int level) {
  unsigned long long code = 0;
  for (int b = 0; b < level; ++b) {
    code |= static_cast<unsigned long long>((ix >> b) & 1) << (3 * b);
    code |= static_cast<unsigned long long>((iy >> b) & 1) << (3 * b + 1);
    code |= static_cast<unsigned long long>((iz >> b) & 1) << (3 * b + 2);
  }
  return code;
}

__global__ void morton_kernel(const double* __restrict__ xyz, std::int64_t n, int cap,
                              unsigned long long* __restrict__ codes,
                              std::int32_t* __restrict__ idx, unsigned* flags) {
  const std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const double x = xyz[3 * i], y = xyz[3 * i + 1], z = xyz[3 * i + 2];
  // domain check (octree.cpp:91-97): lo = -1, hi = lo + 2*half_width = 1
  if (x < -1.0 || x > 1.0 || y < -1.0 || y > 1.0 || z < -1.0 || z > 1.0 || x != x || y != y ||
      z != z)
    atomicOr(flags, kFlagOutOfDomain);
  const long long cells = 1LL << cap;
  codes[i] = morton(grid_coord(x, cells), grid_coord(y, cells), grid_coord(z, cells), cap);
  idx[i] = static_cast<std::int32_t>(i);
}

// first index k in [lo, hi) with codes[k] >= key
__device__ __forceinline__ std::int64_t lower_bound(const unsigned long long* __restrict__ codes,
                                                    std::int64_t lo, std::int64_t hi,
                                                    unsigned long long key) {
  while (lo < hi) {
    const std::int64_t mid = lo + ((hi - lo) >> 1);
    if (codes[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Max occupancy per level (octree.cpp:110-130): every run start measures its
// run by binary search for the next prefix.
__global__ void depth_scan_kernel(const unsigned long long* __restrict__ codes, std::int64_t n,
                                  int cap, unsigned long long* maxocc) {
  const std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const unsigned long long c = codes[i];
  const unsigned long long prev = i > 0 ? codes[i - 1] : ~0ULL;
  for (int l = 0; l <= cap; ++l) {
    const int shift = 3 * (cap - l);
    const unsigned long long pre = c >> shift;
    if (i > 0 && (prev >> shift) == pre) continue;  // not a run start
    std::int64_t end = n;
    if (shift < 64 && pre + 1 <= (~0ULL >> shift)) {
      end = lower_bound(codes, i, n, (pre + 1) << shift);
    }
    atomicMax(&maxocc[l], static_cast<unsigned long long>(end - i));
  }
}

__global__ void node_offsets_kernel(const unsigned long long* __restrict__ codes, std::int64_t n,
                                    int shift, std::int64_t count, std::int64_t* __restrict__ off) {
  const std::int64_t m = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
  if (m > count) return;
  off[m] = m == count ? n : lower_bound(codes, 0, n, static_cast<unsigned long long>(m) << shift);
}

__global__ void permute_kernel(const double* __restrict__ xyz, const std::int32_t* __restrict__ perm,
                               std::int64_t n, double* __restrict__ px, double* __restrict__ py,
                               double* __restrict__ pz) {
  const std::int64_t p = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
  if (p >= n) return;
  const std::int64_t o = perm[p];
  px[p] = xyz[3 * o];
  py[p] = xyz[3 * o + 1];
  pz[p] = xyz[3 * o + 2];
}

inline unsigned grid_for(std::int64_t n, int threads) {
  return static_cast<unsigned>((n + threads - 1) / threads);
}

}  // namespace

void launch_morton_codes(const double* xyz, std::int64_t n, int depth_cap,
                         unsigned long long* codes, std::int32_t* idx, unsigned* flags,
                         cudaStream_t s) {
  morton_kernel<<<grid_for(n, 256), 256, 0, s>>>(xyz, n, depth_cap, codes, idx, flags);
  H3D_CUDA_CHECK(cudaGetLastError());
}

std::size_t radix_sort_temp_bytes(std::int64_t n, int end_bit) {
  std::size_t bytes = 0;
  H3D_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(
      nullptr, bytes, static_cast<const unsigned long long*>(nullptr),
      static_cast<unsigned long long*>(nullptr), static_cast<const std::int32_t*>(nullptr),
      static_cast<std::int32_t*>(nullptr), n, 0, end_bit));
  return bytes;
}

void radix_sort_pairs(void* tmp, std::size_t tmp_bytes, const unsigned long long* kin,
                      unsigned long long* kout, const std::int32_t* vin, std::int32_t* vout,
                      std::int64_t n, int end_bit, cudaStream_t s) {
  H3D_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, kin, kout, vin, vout, n, 0,
                                                 end_bit, s));
}

void launch_depth_scan(const unsigned long long* codes, std::int64_t n, int depth_cap,
                       unsigned long long* maxocc, cudaStream_t s) {
  depth_scan_kernel<<<grid_for(n, 256), 256, 0, s>>>(codes, n, depth_cap, maxocc);
  H3D_CUDA_CHECK(cudaGetLastError());
}

void launch_node_offsets(const unsigned long long* codes, std::int64_t n, int depth_cap,
                         int level, std::int64_t* off, cudaStream_t s) {
  const std::int64_t count = 1LL << (3 * level);
  node_offsets_kernel<<<grid_for(count + 1, 256), 256, 0, s>>>(codes, n, 3 * (depth_cap - level),
                                                              count, off);
  H3D_CUDA_CHECK(cudaGetLastError());
}

void launch_permute_points(const double* xyz, const std::int32_t* perm, std::int64_t n,
                           double* px, double* py, double* pz, cudaStream_t s) {
  permute_kernel<<<grid_for(n, 256), 256, 0, s>>>(xyz, perm, n, px, py, pz);
  H3D_CUDA_CHECK(cudaGetLastError());
}

std::size_t scan_temp_bytes(std::int64_t n) {
  std::size_t bytes = 0;
  H3D_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, bytes,
                                               static_cast<const std::int32_t*>(nullptr),
                                               static_cast<std::int32_t*>(nullptr), n + 1));
  return bytes;
}

void exclusive_scan_i32(void* tmp, std::size_t tmp_bytes, const std::int32_t* in,
                        std::int32_t* out, std::int64_t n, cudaStream_t s) {
  // `in` must have n + 1 entries with in[n] == 0 so out[n] is the total.
  H3D_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, in, out, n + 1, s));
}

}  // namespace h3db
