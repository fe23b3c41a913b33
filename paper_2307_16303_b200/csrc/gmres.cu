// Device-resident GMRES over the HODLR3D operator and the exact dense product
// used to manufacture right-hand sides (reference solver.cpp:22-125 gmres,
// :199-206 IEOperator::apply, :243-300 ie_experiment's dense row sums).
//
// Vectors live in HBM; the Krylov basis is (restart + 1) x N doubles. Every
// reduction is a fixed two-stage tree (kDotBlocks partials, then one block in
// index order), so a solve is bitwise reproducible. The tiny Hessenberg /
// Givens work runs on the host from one (k + 2)-double copy per iteration.
#include "common.cuh"
#include "kernels.h"

namespace h3db {

namespace {

constexpr int kDotBlocks = 296;  // 2 per SM
constexpr int kDotThreads = 256;

__device__ __forceinline__ double block_sum(double v, double* sh) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < kDotThreads / 32; ++w) t += sh[w];
  __syncthreads();
  return t;  // valid in thread 0
}

__global__ void __launch_bounds__(kDotThreads) dot_partial(const double* __restrict__ a,
                                                          const double* __restrict__ b, std::int64_t n,
                                                          double* __restrict__ part) {
  __shared__ double sh[kDotThreads / 32];
  double v = 0.0;
  for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(kDotThreads) + threadIdx.x; i < n;
       i += static_cast<std::int64_t>(kDotBlocks) * kDotThreads)
    v = fma(a[i], b[i], v);
  const double t = block_sum(v, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = t;
}

// out = sum of the partials (index order); mode 1: out = sqrt(sum)
__global__ void __launch_bounds__(kDotThreads) dot_final(const double* __restrict__ part, double* out,
                                                        int mode) {
  __shared__ double sh[kDotThreads / 32];
  double v = 0.0;
  for (int i = threadIdx.x; i < kDotBlocks; i += kDotThreads) v += part[i];
  const double t = block_sum(v, sh);
  if (threadIdx.x == 0) *out = mode == 1 ? sqrt(t) : t;
}

// y += c x, c = sign * (*cdev) (device scalar) or c = chost
__global__ void axpy_kernel(double* __restrict__ y, const double* __restrict__ x, std::int64_t n,
                            const double* cdev, double sign, double chost) {
  const double c = cdev ? sign * *cdev : chost;
  for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
    y[i] = fma(c, x[i], y[i]);
}

// y = x / (*d) (d > 0), else y = x
__global__ void scale_div_kernel(double* __restrict__ y, const double* __restrict__ x, std::int64_t n,
                                 const double* d) {
  const double s = *d;
  for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
    y[i] = s > 0.0 ? x[i] / s : x[i];
}

// w = alpha v + beta w  (the IE operator d I + h^3 K, solver.cpp:199-206)
__global__ void affine_kernel(double* __restrict__ w, const double* __restrict__ v, std::int64_t n,
                              double alpha, double beta) {
  for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
    w[i] = fma(alpha, v[i], beta * w[i]);
}

// r = f - w
__global__ void sub_kernel(double* __restrict__ r, const double* __restrict__ f,
                           const double* __restrict__ w, std::int64_t n) {
  for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
    r[i] = f[i] - w[i];
}

// ---- exact dense product b = K x (diagonal rule), thread per target, sources
// staged in shared memory and read as broadcasts; Morton-order packed points.
template <int K>
__global__ void __launch_bounds__(256) direct_kernel(const double4* __restrict__ p4, std::int64_t n,
                                                     double diag, const std::int32_t* __restrict__ perm,
                                                     double* __restrict__ b) {
  __shared__ double4 src[256];
  const std::int64_t i = blockIdx.x * 256LL + threadIdx.x;
  const double4 t = i < n ? p4[i] : make_double4(1e100, 1e100, 1e100, 0.0);
  double acc0 = 0.0, acc1 = 0.0;
  for (std::int64_t j0 = 0; j0 < n; j0 += 256) {
    __syncthreads();
    if (j0 + threadIdx.x < n) src[threadIdx.x] = p4[j0 + threadIdx.x];
    __syncthreads();
    const int nj = static_cast<int>(n - j0 < 256 ? n - j0 : 256);
    for (int j = 0; j < nj; ++j) {
      const double4 s = src[j];
      const double k = (j0 + j == i) ? diag : kernel_r2_fast<K>(sq3(t.x - s.x, t.y - s.y, t.z - s.z));
      if (j & 1) acc1 = fma(k, s.w, acc1);
      else acc0 = fma(k, s.w, acc0);
    }
  }
  if (i < n) b[perm[i]] = acc0 + acc1;
}

// ---- exact rows for reference_error (reference hmatrix.cpp:253-291): row
// p (Morton position) of K times x, every column, the diagonal rule at j == p
// (KernelBlock with offset 0) and the full-accuracy radial map. One CTA per
// sampled row; fixed-order tree reduction (deterministic). Coincident
// distinct points raise kFlagDegenGeom (lowrank.cpp:34-36).
template <int K>
__global__ void __launch_bounds__(256) exact_rows_kernel(const double4* __restrict__ p4, std::int64_t n,
                                                         double diag, const std::int64_t* __restrict__ rows,
                                                         double* __restrict__ out, unsigned* flags) {
  __shared__ double red[8];
  const std::int64_t p = rows[blockIdx.x];
  const double4 t = p4[p];
  double acc = 0.0;
  bool degen = false;
  for (std::int64_t j = threadIdx.x; j < n; j += 256) {
    const double4 s = p4[j];
    double k;
    if (j == p) {
      k = diag;
    } else {
      const double r2 = sq3(t.x - s.x, t.y - s.y, t.z - s.z);
      degen |= r2 < kCoincidentTol2;
      k = kernel_r2<K>(r2);
    }
    acc = fma(k, s.w, acc);
  }
  if (degen) atomicOr(flags, kFlagDegenGeom);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = 0.0;
    for (int w = 0; w < 8; ++w) v += red[w];
    out[blockIdx.x] = v;
  }
}

unsigned grid1(std::int64_t n) {
  return static_cast<unsigned>(std::min<std::int64_t>((n + 255) / 256, 148 * 16));
}

}  // namespace

std::size_t dot_scratch_doubles() { return kDotBlocks; }

void launch_dot(const double* a, const double* b, std::int64_t n, double* scratch, double* out, bool sqrt_of,
                cudaStream_t s) {
  dot_partial<<<kDotBlocks, kDotThreads, 0, s>>>(a, b, n, scratch);
  dot_final<<<1, kDotThreads, 0, s>>>(scratch, out, sqrt_of ? 1 : 0);
  H3D_CUDA_CHECK(cudaGetLastError());
}

void launch_axpy(double* y, const double* x, std::int64_t n, const double* cdev, double sign, double chost,
                 cudaStream_t s) {
  axpy_kernel<<<grid1(n), 256, 0, s>>>(y, x, n, cdev, sign, chost);
  H3D_CUDA_CHECK(cudaGetLastError());
}

void launch_scale_div(double* y, const double* x, std::int64_t n, const double* d, cudaStream_t s) {
  scale_div_kernel<<<grid1(n), 256, 0, s>>>(y, x, n, d);
  H3D_CUDA_CHECK(cudaGetLastError());
}

void launch_affine(double* w, const double* v, std::int64_t n, double alpha, double beta, cudaStream_t s) {
  affine_kernel<<<grid1(n), 256, 0, s>>>(w, v, n, alpha, beta);
  H3D_CUDA_CHECK(cudaGetLastError());
}

void launch_sub(double* r, const double* f, const double* w, std::int64_t n, cudaStream_t s) {
  sub_kernel<<<grid1(n), 256, 0, s>>>(r, f, w, n);
  H3D_CUDA_CHECK(cudaGetLastError());
}

void launch_direct(const double* p4, std::int64_t n, int kernel, double diag, const std::int32_t* perm,
                   double* b, cudaStream_t s) {
  const unsigned grid = static_cast<unsigned>((n + 255) / 256);
  const double4* q = reinterpret_cast<const double4*>(p4);
  switch (kernel) {
    case kLaplace: direct_kernel<kLaplace><<<grid, 256, 0, s>>>(q, n, diag, perm, b); break;
    case kR4: direct_kernel<kR4><<<grid, 256, 0, s>>>(q, n, diag, perm, b); break;
    default: direct_kernel<kHelmholtz><<<grid, 256, 0, s>>>(q, n, diag, perm, b); break;
  }
  H3D_CUDA_CHECK(cudaGetLastError());
}

void launch_exact_rows(const double* p4, std::int64_t n, int kernel, double diag, const std::int64_t* rows,
                       std::int64_t nrows, double* out, unsigned* flags, cudaStream_t s) {
  const double4* q = reinterpret_cast<const double4*>(p4);
  for (std::int64_t r0 = 0; r0 < nrows; r0 += 65535) {
    const unsigned g = static_cast<unsigned>(std::min<std::int64_t>(65535, nrows - r0));
    switch (kernel) {
      case kLaplace: exact_rows_kernel<kLaplace><<<g, 256, 0, s>>>(q, n, diag, rows + r0, out + r0, flags); break;
      case kR4: exact_rows_kernel<kR4><<<g, 256, 0, s>>>(q, n, diag, rows + r0, out + r0, flags); break;
      default: exact_rows_kernel<kHelmholtz><<<g, 256, 0, s>>>(q, n, diag, rows + r0, out + r0, flags); break;
    }
    H3D_CUDA_CHECK(cudaGetLastError());
  }
}

}  // namespace h3db
