// C++ host layer (include/h3d_b200.hpp): the reference's HODLR3D API over
// the C-ABI of include/h3d_b200.h. Built as lib/libh3d_b200pp.so (g++,
// C++20), linked against lib/libh3d_b200.so; no CUDA or torch types here.
#include "../../include/h3d_b200.hpp"

#include <cmath>
#include <string>

namespace h3d::b200 {

namespace {

// status code -> the reference's exception type (include/h3d_b200.h header)
[[noreturn]] void rethrow(int status) {
  const std::string msg = h3d_last_error();
  switch (status) {
    case H3D_EINVAL:
    case H3D_EUNSUPPORTED:
      throw std::invalid_argument(msg);
    case H3D_EDEGEN_GEOM:
      throw DegenerateGeometryError(msg);
    case H3D_EDEGEN_DIST:
      throw DegenerateDistributionError(msg);
    default:
      throw DeviceError("h3d_b200 status " + std::to_string(status) + ": " + msg);
  }
}

void check(int status) {
  if (status != H3D_OK) rethrow(status);
}

int kernel_code(const KernelSpec& k) {
  switch (k.id) {
    case KernelId::Laplace3d: return H3D_LAPLACE3D;
    case KernelId::InverseQuartic: return H3D_R4;
    case KernelId::HelmholtzRe: return H3D_HELMHOLTZ_RE;
    case KernelId::Custom: break;
  }
  throw std::invalid_argument("initialize: custom std::function kernels cannot run on the device");
}

}  // namespace

// kernel.cpp:7-21
double KernelSpec::operator()(double r) const {
  switch (id) {
    case KernelId::Laplace3d: return 1.0 / r;
    case KernelId::InverseQuartic: {
      const double r2 = r * r;
      return 1.0 / (r2 * r2);
    }
    case KernelId::HelmholtzRe: return std::cos(r) / r;
    case KernelId::Custom: break;
  }
  throw std::invalid_argument("custom kernels are not supported by the device engine");
}

// kernel.cpp:23-41
KernelSpec make_kernel(KernelId id) {
  KernelSpec k;
  k.id = id;
  switch (id) {
    case KernelId::Laplace3d: k.name = "laplace3d"; break;
    case KernelId::InverseQuartic: k.name = "r4"; break;
    case KernelId::HelmholtzRe: k.name = "helmholtz-re"; break;
    case KernelId::Custom: throw std::invalid_argument("custom kernels cannot run on the device");
  }
  return k;
}

// kernel.cpp:52-57
KernelSpec parse_kernel(const std::string& name) {
  if (name == "laplace3d") return make_kernel(KernelId::Laplace3d);
  if (name == "r4") return make_kernel(KernelId::InverseQuartic);
  if (name == "helmholtz-re") return make_kernel(KernelId::HelmholtzRe);
  throw std::invalid_argument("unknown kernel: " + name);
}

// kernel.cpp:82-112 (h3d_generate_points / h3d_generate_grid_points are
// bit-identical to it)
PointSet generate_points(Distribution dist, std::size_t n, std::uint64_t seed) {
  if (n < 1) throw std::invalid_argument("generate_points: N must be >= 1");
  PointSet ps;
  ps.seed = seed;
  ps.distribution = dist;
  ps.points.resize(n);
  double* xyz = &ps.points[0].x;  // Point3 is three packed doubles: AoS xyz[3n]
  static_assert(sizeof(Point3) == 3 * sizeof(double), "Point3 must be packed");
  if (dist == Distribution::UniformRandom)
    check(h3d_generate_points(static_cast<std::int64_t>(n), seed, xyz));
  else
    check(h3d_generate_grid_points(static_cast<std::int64_t>(n), xyz));
  return ps;
}

// hmatrix.cpp:52-151
HMatrixRep initialize(const PointSet& pts, const KernelSpec& kernel, Variant variant, const HmatOptions& o) {
  if (pts.size() == 0) throw std::invalid_argument("initialize: empty point set");
  return initialize(&pts.points[0].x, pts.size(), kernel, variant, o);
}

HMatrixRep initialize(const double* xyz, std::size_t n, const KernelSpec& kernel, Variant variant,
                      const HmatOptions& o) {
  if (n == 0 || xyz == nullptr) throw std::invalid_argument("initialize: empty point set");
  if (!(o.epsilon > 0.0)) throw std::invalid_argument("initialize: epsilon must be positive");
  h3d_options opt;
  h3d_default_options(&opt);
  opt.kernel_id = kernel_code(kernel);
  opt.diagonal = kernel.diagonal;
  opt.n_max = o.n_max;
  opt.epsilon = o.epsilon;
  opt.depth_cap = o.depth_cap;
  opt.max_rank = o.max_rank;
  opt.near_mode = o.dense_mode == DenseMode::Cached ? H3D_NEAR_STORED : H3D_NEAR_MATRIX_FREE;
  opt.device = o.device;
  opt.mode_policy = o.mode_policy;
  opt.gather_b = o.gather_b;
  opt.variant = static_cast<int>(variant);
  h3d_dev* dev = nullptr;
  check(h3d_dev_create(xyz, static_cast<std::int64_t>(n), &opt, &dev));
  HMatrixRep rep;
  rep.dev_ = std::shared_ptr<h3d_dev>(dev, [](h3d_dev* d) { h3d_dev_destroy(d); });
  rep.variant = variant;
  rep.kernel = kernel;
  rep.options = o;
  rep.n_ = n;
  h3d_stats st{};
  check(h3d_dev_stats(dev, &st));
  rep.depth_ = st.depth;
  return rep;
}

// hmatrix.cpp:153-226
std::vector<double> matvec(const HMatrixRep& rep, std::span<const double> x, MatvecTiming* timing) {
  if (!rep.handle()) throw std::invalid_argument("matvec: uninitialised representation");
  if (x.size() != rep.n()) throw std::invalid_argument("matvec: vector length != N");
  std::vector<double> b(rep.n());
  h3d_timing t{};
  check(h3d_dev_matvec(rep.handle(), x.data(), b.data(), /*host*/ 0, timing ? &t : nullptr));
  if (timing) {
    timing->wall_seconds = t.total_ms * 1e-3;
    timing->dense_gen_seconds = 0.0;
    timing->matvec_seconds = t.total_ms * 1e-3;
  }
  return b;
}

// hmatrix.cpp:228-251
RepStats stats(const HMatrixRep& rep) {
  if (!rep.handle()) throw std::invalid_argument("stats: uninitialised representation");
  h3d_stats st{};
  check(h3d_dev_stats(rep.handle(), &st));
  RepStats s;
  s.float_count = st.ref_float_count;
  s.int_count = st.ref_int_count;
  s.memory_bytes = 8 * s.float_count + 4 * s.int_count;
  s.compression_ratio = st.compression_ratio;
  s.max_rank = st.max_rank;
  s.depth = st.depth;
  s.init_seconds = st.build_ms_total * 1e-3;
  s.dense_form_seconds = 0.0;
  return s;
}

// hmatrix.cpp:253-291
double reference_error(const HMatrixRep& rep, std::span<const double> x, std::span<const double> b_approx,
                       std::size_t exact_limit, std::size_t sample_rows, std::uint64_t seed) {
  if (!rep.handle()) throw std::invalid_argument("reference_error: uninitialised representation");
  if (x.size() != rep.n() || b_approx.size() != rep.n())
    throw std::invalid_argument("reference_error: length mismatch");
  double out = 0.0;
  check(h3d_dev_reference_error(rep.handle(), x.data(), b_approx.data(), /*host*/ 0,
                                static_cast<std::int64_t>(exact_limit), static_cast<std::int64_t>(sample_rows),
                                seed, &out));
  return out;
}

}  // namespace h3d::b200
