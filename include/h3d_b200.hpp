// h3d_b200.hpp — C++ host layer of the B200 HODLR3D engine.
//
// The reference's operator surface for this path, kept signature for
// signature (reference proj/include/h3d/kernel.hpp, octree.hpp, hmatrix.hpp):
//
//   PointSet     generate_points(Distribution, N, seed)          kernel.hpp:38
//   KernelSpec   make_kernel(KernelId) / parse_kernel(name)      kernel.hpp:55-59
//   HMatrixRep   initialize(pts, kernel, variant, HmatOptions)   hmatrix.hpp:57-58
//   std::vector<double> matvec(rep, x, MatvecTiming*)            hmatrix.hpp:70-71
//   RepStats     stats(rep)                                      hmatrix.hpp:85
//   double       reference_error(rep, x, b, 4096, 2000, 7)       hmatrix.hpp:90-93
//
// in namespace h3d::b200, over the C-ABI of include/h3d_b200.h (the library
// lib/libh3d_b200.so; this layer is lib/libh3d_b200pp.so). Every call runs on
// the GPU: there is no CPU fallback. Errors are the reference's exceptions:
// std::invalid_argument (bad arguments, length mismatch, custom std::function
// kernels — they cannot cross to the device), DegenerateGeometryError,
// DegenerateDistributionError; device failures raise DeviceError
// (a std::runtime_error).
//
// HMatrixRep owns the device representation through a shared handle: copies
// share it, it is immutable after initialize(), and concurrent matvec() calls
// from several threads are safe (the handle serialises them, the results are
// bitwise deterministic — reference hmatrix.hpp:34-36, 68-69).
#pragma once

#include <cstddef>
#include <cstdint>
#include <memory>
#include <random>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "h3d_b200.h"

namespace h3d::b200 {

// ---- kernel.hpp
struct Point3 {
  double x = 0.0, y = 0.0, z = 0.0;
};

/// Top 53 bits of the engine output (reference kernel.hpp:24-26).
inline double uniform01(std::mt19937_64& gen) { return static_cast<double>(gen() >> 11) * 0x1.0p-53; }

enum class Distribution { UniformRandom, TensorGrid };

struct PointSet {
  std::vector<Point3> points;
  std::uint64_t seed = 0;
  Distribution distribution = Distribution::UniformRandom;
  std::size_t size() const { return points.size(); }
};

/// Bit-identical to the reference generators (kernel.cpp:88-109).
PointSet generate_points(Distribution dist, std::size_t n, std::uint64_t seed);

enum class KernelId { Laplace3d, InverseQuartic, HelmholtzRe, Custom };

struct KernelSpec {
  KernelId id = KernelId::Laplace3d;
  std::string name = "laplace3d";
  double diagonal = 0.0;
  /// f(r) of the built-in kernels (host evaluation, kernel.cpp:7-21)
  double operator()(double r) const;
};

KernelSpec make_kernel(KernelId id);
/// "laplace3d", "r4", "helmholtz-re" (kernel.cpp:52-57)
KernelSpec parse_kernel(const std::string& name);

struct DegenerateGeometryError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ---- octree.hpp
struct DegenerateDistributionError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

enum class Variant { Hodlr3d, Hodlr, HStrong };

// ---- hmatrix.hpp
enum class DenseMode { OnTheFly, Cached };

struct HmatOptions {
  int n_max = 216;
  double epsilon = 1e-7;
  DenseMode dense_mode = DenseMode::OnTheFly;
  int depth_cap = 12;
  std::int64_t max_rank = 0;  // 0: min(|X|,|Y|) per block
  // B200 extensions (not in the reference struct): CUDA device ordinal and
  // the per-level representation policy (h3d_options.mode_policy: 0 stream,
  // 1 auto, 2 explicit level_modes).
  int device = 0;
  int mode_policy = 1;
  int gather_b = 0;  // multi-GPU: every rank returns the full b (h3d_options.gather_b)
};

/// Raised on CUDA / NCCL / allocation failures inside the engine.
struct DeviceError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

class HMatrixRep {
 public:
  Variant variant = Variant::Hodlr3d;
  KernelSpec kernel;
  HmatOptions options;

  std::size_t n() const { return n_; }
  int depth() const { return depth_; }
  /// the C-ABI handle (for h3d_dev_matvec_async, profiling, GMRES)
  h3d_dev* handle() const { return dev_.get(); }

 private:
  friend HMatrixRep initialize(const double*, std::size_t, const KernelSpec&, Variant, const HmatOptions&);
  std::shared_ptr<h3d_dev> dev_;
  std::size_t n_ = 0;
  int depth_ = 0;
};

HMatrixRep initialize(const PointSet& pts, const KernelSpec& kernel, Variant variant,
                      const HmatOptions& options = {});
/// The same from an AoS coordinate array xyz[3n] (any Point3-compatible
/// storage, e.g. the reference's own PointSet::points).
HMatrixRep initialize(const double* xyz, std::size_t n, const KernelSpec& kernel, Variant variant,
                      const HmatOptions& options = {});

struct MatvecTiming {
  double wall_seconds = 0.0;
  double dense_gen_seconds = 0.0;  // 0: the near field is generated inside the matvec kernels
  double matvec_seconds = 0.0;
};

/// b = A~ x in the original point order.
std::vector<double> matvec(const HMatrixRep& rep, std::span<const double> x, MatvecTiming* timing = nullptr);

struct RepStats {
  std::uint64_t float_count = 0;  // r^2 per ordered block + dense leaf areas
  std::uint64_t int_count = 0;    // pivot indices
  std::uint64_t memory_bytes = 0;
  double compression_ratio = 0.0;
  int max_rank = 0;
  int depth = 0;
  double init_seconds = 0.0;
  double dense_form_seconds = 0.0;
  double matvec_seconds = 0.0;  // filled by the harness
};

RepStats stats(const HMatrixRep& rep);

double reference_error(const HMatrixRep& rep, std::span<const double> x, std::span<const double> b_approx,
                       std::size_t exact_limit = 4096, std::size_t sample_rows = 2000, std::uint64_t seed = 7);

}  // namespace h3d::b200
