// h3d_b200_ref.hpp — drop-in binding for code written against the
// reference's own types (proj/include/h3d/*.hpp). Header-only; include it
// after the reference headers:
//
//   #include "h3d/hmatrix.hpp"     // reference: PointSet, KernelSpec, Variant, HmatOptions
//   #include "h3d_b200_ref.hpp"    // this file
//
//   h3d::b200::HMatrixRep rep = h3d::b200::initialize(pts, kernel, h3d::Variant::Hodlr3d, opt);
//   std::vector<double> b = h3d::b200::matvec(rep, x);            // hmatrix.hpp:70-71
//   h3d::RepStats st = h3d::b200::reference_stats(rep);           // hmatrix.hpp:85
//   double err = h3d::b200::reference_error(rep, x, b);           // hmatrix.hpp:90-93
//
// Exceptions come back as the reference's types (h3d::DegenerateGeometryError,
// kernel.hpp:64-66; h3d::DegenerateDistributionError, octree.hpp:41-43;
// std::invalid_argument). The reference's Point3 is three packed doubles, so
// its PointSet storage is passed to the device without a copy. Link
// lib/libh3d_b200pp.so and lib/libh3d_b200.so.
#pragma once

#include "h3d_b200.hpp"

namespace h3d::b200 {

static_assert(sizeof(h3d::Point3) == 3 * sizeof(double), "reference Point3 must be three packed doubles");

inline KernelSpec from_reference(const h3d::KernelSpec& k) {
  if (k.id == h3d::KernelId::Custom)
    throw std::invalid_argument("custom std::function kernels (kernel.hpp:56-57) cannot run on the device");
  KernelSpec out = make_kernel(static_cast<KernelId>(static_cast<int>(k.id)));
  out.diagonal = k.diagonal;
  return out;
}

inline HmatOptions from_reference(const h3d::HmatOptions& o, int device = 0) {
  HmatOptions out;
  out.n_max = o.n_max;
  out.epsilon = o.epsilon;
  out.dense_mode = o.dense_mode == h3d::DenseMode::Cached ? DenseMode::Cached : DenseMode::OnTheFly;
  out.depth_cap = o.depth_cap;
  out.max_rank = o.max_rank;
  out.device = device;
  return out;
}

/// hmatrix.hpp:57-58 on the reference's argument types.
inline HMatrixRep initialize(const h3d::PointSet& pts, const h3d::KernelSpec& kernel, h3d::Variant variant,
                             const h3d::HmatOptions& options = {}, int device = 0) {
  try {
    return initialize(pts.size() ? &pts.points[0].x : nullptr, pts.size(), from_reference(kernel),
                      static_cast<Variant>(static_cast<int>(variant)), from_reference(options, device));
  } catch (const DegenerateGeometryError& e) {
    throw h3d::DegenerateGeometryError(e.what());
  } catch (const DegenerateDistributionError& e) {
    throw h3d::DegenerateDistributionError(e.what());
  }
}

/// hmatrix.hpp:85 as the reference's RepStats.
inline h3d::RepStats reference_stats(const HMatrixRep& rep) {
  const RepStats s = stats(rep);
  h3d::RepStats r;
  r.float_count = s.float_count;
  r.int_count = s.int_count;
  r.memory_bytes = s.memory_bytes;
  r.compression_ratio = s.compression_ratio;
  r.max_rank = s.max_rank;
  r.depth = s.depth;
  r.init_seconds = s.init_seconds;
  r.dense_form_seconds = s.dense_form_seconds;
  return r;
}

}  // namespace h3d::b200
