// Shared device helpers for the B200 HODLR3D engine (sm_100a only).
#pragma once

#include <cstdint>
#include <mutex>
#include <cuda_runtime.h>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "h3d_b200 targets sm_100a only"
#endif

namespace h3db {

// Kernel ids follow h3d::KernelId (reference kernel.hpp:42).
enum KernelKind : int { kLaplace = 0, kR4 = 1, kHelmholtz = 2 };

// Device status flags (bitwise OR'ed by kernels, read by the host).
enum DevFlag : unsigned {
  kFlagDegenGeom = 1u,    // r < 1e-14 between distinct points (kernel.cpp:59-71)
  kFlagAcaOverflow = 2u,  // ACA workspace rank capacity exhausted
  kFlagOutOfDomain = 4u,  // point outside [-1,1]^3 (octree.cpp:91-97)
  kFlagPoolFull = 8u,     // single-pass ACA: the rank pass's LU pool is exhausted
};

constexpr double kCoincidentTol2 = 1e-14 * 1e-14;

// Radial map on r^2 (reference lowrank.cpp:51-62: LaplaceF, QuarticF,
// HelmholtzF). Laplace uses the fp64 reciprocal square root (<= 1 ulp from
// 1/sqrt(r2)); parity is tolerance-based (north_star: 10x ACA tol).
template <int K>
__device__ __forceinline__ double kernel_r2(double r2) {
  if constexpr (K == kLaplace) {
    return rsqrt(r2);
  } else if constexpr (K == kR4) {
    return 1.0 / (r2 * r2);
  } else {
    const double r = sqrt(r2);
    return cos(r) / r;
  }
}

// Matvec-path radial map: Laplace uses the hardware fp64 rsqrt seed
// (MUFU.RSQ64H, ~2^-22) plus one third-order correction
//   y1 = y0 (1 + e/2 + 3e^2/8),  e = 1 - x y0^2,
// cubic convergence: full double accuracy (the depth-0 dense matvec matches the
// direct sum to < 1e-13, reference test_hmatrix.cpp:21-35) for 5 FP64 ops,
// cheaper than rsqrt()'s two Newton steps + special-case handling.
__device__ __forceinline__ double rsqrt_c3(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double p = x * y;
  const double e = fma(-p, y, 1.0);
  const double c = fma(e, 0.375, 0.5);
  return fma(y, e * c, y);
}

// Admissible-block evaluations (proxy regeneration, direct leaf blocks):
// one Newton step from the same seed, with the factor -1/2 folded out of the
// sum:  1/sqrt(x) ~= -0.5 * y0 (x y0^2 - 3)  (relative error ~1e-13, far
// below any ACA tolerance these blocks are compressed or compared at), i.e.
// acc += y0 (x y0^2 - 3) w costs 4 FP64 ops after the seed; the caller scales
// its accumulator by kNewtonScale once.
constexpr double kNewtonScale = -0.5;
__device__ __forceinline__ double rsqrt_n1_acc(double x, double w, double acc) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double t = x * y;
  const double h = fma(t, y, -3.0);
  return fma(y * h, w, acc);
}

// acc += K(r2) w on the admissible path (Laplace: Newton form, scaled later
// by far_scale<K>(); others exact)
// 1/r^4 = (1/r)^4 from the same Newton form: g = y0 (x y0^2 - 3) = -2/r,
// so g^4 = 16 / r^4 (scale 1/16), no division.
__device__ __forceinline__ double rsqrt4_n1_acc(double x, double w, double acc) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double t = x * y;
  const double g = y * fma(t, y, -3.0);
  const double g2 = g * g;
  return fma(g2 * g2, w, acc);
}

template <int K>
__device__ __forceinline__ double far_acc(double r2, double w, double acc) {
  if constexpr (K == kLaplace) {
    return rsqrt_n1_acc(r2, w, acc);
  } else if constexpr (K == kR4) {
    return rsqrt4_n1_acc(r2, w, acc);
  } else {
    return fma(kernel_r2<K>(r2), w, acc);
  }
}
// the admissible-path value itself, far_scale-scaled like far_acc (no
// accumulate: one FP64 instruction fewer than far_acc(r2, 1.0, 0.0))
template <int K>
__device__ __forceinline__ double far_val(double r2) {
  if constexpr (K == kLaplace || K == kR4) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r2));
    const double g = y * fma(r2 * y, y, -3.0);
    if constexpr (K == kLaplace) {
      return g;
    } else {
      const double g2 = g * g;
      return g2 * g2;
    }
  } else {
    return kernel_r2<K>(r2);
  }
}

template <int K>
__device__ __forceinline__ constexpr double far_scale() {
  return K == kLaplace ? kNewtonScale : K == kR4 ? 1.0 / 16.0 : 1.0;
}

template <int K>
__device__ __forceinline__ double kernel_r2_fast(double r2) {
  if constexpr (K == kLaplace) {
    return rsqrt_c3(r2);
  } else if constexpr (K == kR4) {
    const double y = rsqrt_c3(r2);
    const double y2 = y * y;
    return y2 * y2;
  } else {
    return kernel_r2<K>(r2);
  }
}

__device__ __forceinline__ double sq3(double dx, double dy, double dz) {
  return fma(dz, dz, fma(dy, dy, dx * dx));
}

// Deterministic warp reductions (fixed butterfly order).
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// argmax with ties to the lowest index; idx < 0 means "no candidate".
__device__ __forceinline__ void argmax_combine(double& v, long long& i, double v2,
                                               long long i2) {
  if (i2 >= 0 && (i < 0 || v2 > v || (v2 == v && i2 < i))) {
    v = v2;
    i = i2;
  }
}

__device__ __forceinline__ void warp_argmax(double& v, long long& i) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
    const long long i2 = __shfl_xor_sync(0xffffffffu, i, o);
    argmax_combine(v, i, v2, i2);
  }
}

__device__ __forceinline__ long long warp_min_ll(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const long long v2 = __shfl_xor_sync(0xffffffffu, v, o);
    v = v2 < v ? v2 : v;
  }
  return v;
}

// Streaming 16-byte load that bypasses L1 allocation (factor pools are read
// once per matvec phase and are far larger than L2).
__device__ __forceinline__ double2 ld_stream(const double2* p) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
               : "=d"(r.x), "=d"(r.y)
               : "l"(p));
  return r;
}

// The same as a plain (non-volatile) asm: read-only data the compiler may
// batch and schedule freely (stored near-field values).
__device__ __forceinline__ double ldg_stream(const double* p) {
  double r;
  asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(r) : "l"(p));
  return r;
}

__device__ __forceinline__ double ld_stream1(const double* p) {
  double r;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(r) : "l"(p));
  return r;
}

// ---- bulk-copy pipeline primitives (TMA engine, sm_90+ PTX; sm_100a here)
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
// Waits for the phase with the given parity. Between probes the warp sleeps
// (growing backoff): the pipeline kernels share SMs with FP64-bound kernels
// and a spinning waiter would take their issue slots.
__device__ __forceinline__ bool mbar_try(unsigned long long* b, unsigned parity) {
  unsigned done;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}"
      : "=r"(done)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return done != 0;
}
// Every device-side wait is bounded: a wait that outlives H3D_WAIT_LIMIT_NS
// (a pipeline protocol fault, never a slow copy) traps, so the host sees a
// launch failure (H3D_ECUDA) instead of a hung stream.
#ifndef H3D_WAIT_LIMIT_NS
#define H3D_WAIT_LIMIT_NS 20000000000ULL
#endif
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  if (mbar_try(b, parity)) return;
  const unsigned long long t0 = global_ns();
  for (unsigned k = 1;; ++k) {
    if (mbar_try(b, parity)) return;
    if ((k & 1023u) == 0 && global_ns() - t0 > H3D_WAIT_LIMIT_NS) __trap();
  }
}
__device__ __forceinline__ unsigned long long l2_evict_first() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ unsigned long long l2_evict_last() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// global -> shared bulk copy (16-B aligned, multiple of 16 bytes), completion
// counted in bytes on the stage's mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar, unsigned long long pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void named_bar(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// Host: run f() once per (flag, current device). Function attributes
// (dynamic shared memory, carveout) are per device, and one process may drive
// engines on several GPUs.
struct PerDeviceOnce {
  std::mutex mu;
  unsigned long long seen = 0;
  template <class F>
  void operator()(F&& f) {
    int d = 0;
    cudaGetDevice(&d);
    const unsigned long long bit = 1ull << (d & 63);
    std::lock_guard<std::mutex> g(mu);
    if (seen & bit) return;
    f();
    seen |= bit;
  }
};

}  // namespace h3db

#define H3D_CUDA_CHECK(expr)                                                   \
  do {                                                                         \
    cudaError_t e_ = (expr);                                                   \
    if (e_ != cudaSuccess) {                                                   \
      cudaGetLastError(); /* clear a non-sticky error so later checks see their own */ \
      throw ::h3db::CudaError(e_, #expr, __FILE__, __LINE__);                  \
    }                                                                          \
  } while (0)
