// TEST INFRASTRUCTURE ONLY (oracle/): a flat extern "C" wrapper around the
// UNMODIFIED reference library (/root/reference/proj/src/*.cpp compiled in
// place against oracle/shim, see oracle/Makefile). It is the checker and the
// CPU baseline ("kind": "reference"): tests/, __graft_entry__.smoke() and
// bench.py's reference leg load oracle/_ref/libh3dref.so through ctypes.
// Nothing here is linked into the product library.
//
// Every entry point catches the reference's exceptions and reports them as a
// status code plus a message (h3dref_last_error), mirroring the product
// C-ABI's error convention (include/h3d_b200.h).
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include <omp.h>

#include "h3d/hmatrix.hpp"
#include "h3d/parallel.hpp"
#include "h3d/solver.hpp"

using namespace h3d;

namespace {

thread_local std::string g_err;

enum Status : int {
  kOk = 0,
  kInvalid = 1,       // std::invalid_argument
  kDegenGeom = 2,     // DegenerateGeometryError
  kDegenDist = 3,     // DegenerateDistributionError
  kRuntime = 4,       // other std::exception
};

template <class F>
int guarded(F&& f) {
  try {
    f();
    return kOk;
  } catch (const DegenerateGeometryError& e) {
    g_err = e.what();
    return kDegenGeom;
  } catch (const DegenerateDistributionError& e) {
    g_err = e.what();
    return kDegenDist;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return kInvalid;
  } catch (const std::exception& e) {
    g_err = e.what();
    return kRuntime;
  }
}

KernelSpec kernel_of(int id, double diag) {
  KernelSpec k = make_kernel(static_cast<KernelId>(id));
  k.diagonal = diag;
  return k;
}

PointSet pointset_of(const double* xyz, std::int64_t n) {
  PointSet ps;
  ps.points.resize(static_cast<std::size_t>(n));
  std::memcpy(ps.points.data(), xyz, sizeof(double) * 3 * static_cast<std::size_t>(n));
  return ps;
}

struct RefHandle {
  HMatrixRep rep;
};

}  // namespace

extern "C" {

const char* h3dref_last_error(void) { return g_err.c_str(); }

void h3dref_set_threads(int n) {
  if (n > 0) omp_set_num_threads(n);
}
int h3dref_max_threads(void) { return omp_get_max_threads(); }

// kernel.cpp:88-112
int h3dref_generate_points(int dist, std::int64_t n, std::uint64_t seed, double* out_xyz) {
  return guarded([&] {
    const PointSet ps = generate_points(static_cast<Distribution>(dist),
                                        static_cast<std::size_t>(n), seed);
    std::memcpy(out_xyz, ps.points.data(), sizeof(double) * 3 * ps.size());
  });
}

// The CLI/test right-hand side: mt19937_64(seed), 2u-1 (tools/h3d.cpp:135-137).
void h3dref_random_vector(std::int64_t n, std::uint64_t seed, double* out) {
  std::mt19937_64 gen(seed);
  for (std::int64_t i = 0; i < n; ++i) out[i] = 2.0 * uniform01(gen) - 1.0;
}

// hmatrix.cpp:52-151
int h3dref_initialize(const double* xyz, std::int64_t n, int kernel_id, double diag,
                      int variant, int n_max, double eps, int dense_mode, int depth_cap,
                      std::int64_t max_rank, void** out) {
  *out = nullptr;
  return guarded([&] {
    const PointSet ps = pointset_of(xyz, n);
    HmatOptions opt;
    opt.n_max = n_max;
    opt.epsilon = eps;
    opt.dense_mode = dense_mode ? DenseMode::Cached : DenseMode::OnTheFly;
    opt.depth_cap = depth_cap;
    opt.max_rank = max_rank;
    auto h = std::make_unique<RefHandle>();
    h->rep = initialize(ps, kernel_of(kernel_id, diag), static_cast<Variant>(variant), opt);
    *out = h.release();
  });
}

// octree.cpp:76-171 + 197-260 only (no ACA): the tree and lists of a large
// configuration for the bit-exact digest (tests/golden/make_golden_large.py)
int h3dref_tree_lists(const double* xyz, std::int64_t n, int n_max, int variant, void** out) {
  *out = nullptr;
  return guarded([&] {
    const PointSet ps = pointset_of(xyz, n);
    auto h = std::make_unique<RefHandle>();
    h->rep.variant = static_cast<Variant>(variant);
    h->rep.tree = build_tree(ps, n_max);
    h->rep.lists = build_interaction_lists(h->rep.tree, h->rep.variant);
    *out = h.release();
  });
}

void h3dref_free(void* h) { delete static_cast<RefHandle*>(h); }

// hmatrix.cpp:153-226; timing = {wall, dense_gen, matvec_seconds}
int h3dref_matvec(void* h, const double* x, double* b, double* timing3) {
  return guarded([&] {
    const auto& rep = static_cast<RefHandle*>(h)->rep;
    MatvecTiming t;
    const auto out = matvec(rep, std::span<const double>(x, rep.n()), &t);
    std::memcpy(b, out.data(), sizeof(double) * out.size());
    if (timing3) {
      timing3[0] = t.wall_seconds;
      timing3[1] = t.dense_gen_seconds;
      timing3[2] = t.matvec_seconds;
    }
  });
}

// parallel.cpp:111-306
int h3dref_parallel_matvec(void* h, const double* x, int n_p, double* b,
                           std::uint64_t* ledger3) {
  return guarded([&] {
    const auto& rep = static_cast<RefHandle*>(h)->rep;
    const auto res = parallel_matvec(rep, std::span<const double>(x, rep.n()), n_p);
    std::memcpy(b, res.b.data(), sizeof(double) * res.b.size());
    if (ledger3) {
      ledger3[0] = res.ledger.lowrank_exchange_floats;
      ledger3[1] = res.ledger.final_gather_floats;
      ledger3[2] = res.ledger.gather_ops;
    }
  });
}

// hmatrix.cpp:253-291
int h3dref_reference_error(void* h, const double* x, const double* b, double* out) {
  return guarded([&] {
    const auto& rep = static_cast<RefHandle*>(h)->rep;
    *out = reference_error(rep, std::span<const double>(x, rep.n()),
                           std::span<const double>(b, rep.n()));
  });
}

// hmatrix.cpp:228-251; out = {float_count, int_count, memory_bytes, max_rank, depth}
void h3dref_stats(void* h, std::uint64_t* out5, double* secs3) {
  const auto& rep = static_cast<RefHandle*>(h)->rep;
  const RepStats s = stats(rep);
  out5[0] = s.float_count;
  out5[1] = s.int_count;
  out5[2] = s.memory_bytes;
  out5[3] = static_cast<std::uint64_t>(s.max_rank);
  out5[4] = static_cast<std::uint64_t>(s.depth);
  if (secs3) {
    secs3[0] = rep.init_seconds;
    secs3[1] = rep.aca_seconds;
    secs3[2] = rep.dense_form_seconds;
  }
}

int h3dref_depth(void* h) { return static_cast<RefHandle*>(h)->rep.tree.depth; }

// octree.hpp:56-68: perm (permuted position -> original index)
void h3dref_export_perm(void* h, std::int32_t* perm) {
  const auto& t = static_cast<RefHandle*>(h)->rep.tree;
  std::memcpy(perm, t.perm.data(), sizeof(std::int32_t) * t.perm.size());
}

// levels[l][m] = {begin, end}; out has 2 * 8^l int64
void h3dref_export_ranges(void* h, int level, std::int64_t* out) {
  const auto& t = static_cast<RefHandle*>(h)->rep.tree;
  const auto& lv = t.levels[static_cast<std::size_t>(level)];
  for (std::size_t m = 0; m < lv.size(); ++m) {
    out[2 * m] = lv[m].begin;
    out[2 * m + 1] = lv[m].end;
  }
}

// kind: 0 inter, 1 near_edge, 2 near_face, 3 near_vertex. If ids == nullptr
// only offsets (8^l + 1 entries) are written; returns the total count.
std::int64_t h3dref_export_list(void* h, int level, int kind, std::int32_t* offsets,
                                std::int32_t* ids) {
  const auto& L = static_cast<RefHandle*>(h)->rep.lists.levels[static_cast<std::size_t>(level)];
  std::int64_t total = 0;
  for (std::size_t m = 0; m < L.size(); ++m) {
    const NodeLists& nl = L[m];
    const std::vector<std::int32_t>& v =
        kind == 0 ? nl.inter : kind == 1 ? nl.near_edge : kind == 2 ? nl.near_face : nl.near_vertex;
    if (offsets) offsets[m] = static_cast<std::int32_t>(total);
    if (ids) std::memcpy(ids + total, v.data(), sizeof(std::int32_t) * v.size());
    total += static_cast<std::int64_t>(v.size());
  }
  if (offsets) offsets[L.size()] = static_cast<std::int32_t>(total);
  return total;
}

// lr_levels[l]: (target, source, rank) per block, in the reference's order.
std::int64_t h3dref_lr_blocks(void* h, int level, std::int32_t* target, std::int32_t* source,
                              std::int32_t* rank) {
  const auto& v = static_cast<RefHandle*>(h)->rep.lr_levels[static_cast<std::size_t>(level)];
  if (target) {
    for (std::size_t k = 0; k < v.size(); ++k) {
      target[k] = v[k].target;
      source[k] = v[k].source;
      rank[k] = v[k].block.rank();
    }
  }
  return static_cast<std::int64_t>(v.size());
}

// Pivots and packed LU (row-major r x r) of one low-rank block.
void h3dref_lr_block_detail(void* h, int level, std::int64_t k, std::int32_t* row_piv,
                            std::int32_t* col_piv, double* lu) {
  const auto& e = static_cast<RefHandle*>(h)->rep.lr_levels[static_cast<std::size_t>(level)]
                      [static_cast<std::size_t>(k)];
  const int r = e.block.rank();
  for (int a = 0; a < r; ++a) {
    row_piv[a] = e.block.row_pivots[static_cast<std::size_t>(a)];
    col_piv[a] = e.block.col_pivots[static_cast<std::size_t>(a)];
    for (int b = 0; b < r; ++b) lu[a * r + b] = e.block.lu(a, b);
  }
}

// Dense leaf blocks (target, source, class) in matvec visit order.
std::int64_t h3dref_dense_blocks(void* h, std::int32_t* target, std::int32_t* source,
                                 std::int32_t* cls) {
  const auto& v = static_cast<RefHandle*>(h)->rep.dense_blocks;
  if (target) {
    for (std::size_t k = 0; k < v.size(); ++k) {
      target[k] = v[k].target;
      source[k] = v[k].source;
      cls[k] = static_cast<std::int32_t>(v[k].cls);
    }
  }
  return static_cast<std::int64_t>(v.size());
}

// Standalone ACA on one kernel block between two point arrays
// (lowrank.cpp:157-289). Returns the rank; pivots/LU written when room.
int h3dref_aca_block(const double* xs, std::int64_t m, const double* ys, std::int64_t n,
                     int kernel_id, double eps, std::int64_t max_rank, std::int32_t* row_piv,
                     std::int32_t* col_piv, double* lu, std::int64_t cap, int* rank_out) {
  return guarded([&] {
    const KernelSpec k = kernel_of(kernel_id, 0.0);
    const KernelBlock block(k, reinterpret_cast<const Point3*>(xs), m,
                            reinterpret_cast<const Point3*>(ys), n);
    AcaOptions opt;
    opt.epsilon = eps;
    opt.max_rank = max_rank;
    const LowRankBlock lr = aca_compress(block, opt);
    const int r = lr.rank();
    *rank_out = r;
    if (r <= cap) {
      for (int a = 0; a < r; ++a) {
        row_piv[a] = lr.row_pivots[static_cast<std::size_t>(a)];
        col_piv[a] = lr.col_pivots[static_cast<std::size_t>(a)];
        for (int b = 0; b < r; ++b) lu[a * r + b] = lr.lu(a, b);
      }
    }
  });
}

// Census totals (octree.cpp:262-319): {dense, lowrank, ws, vertex, edge, face,
// coverage_area, n_squared}
void h3dref_census(void* h, std::uint64_t* out8) {
  const auto& rep = static_cast<RefHandle*>(h)->rep;
  const BlockCensus c = census(rep.tree, rep.lists);
  out8[0] = c.dense_total;
  out8[1] = c.lowrank_total;
  out8[2] = c.lowrank_ws;
  out8[3] = c.lowrank_vertex;
  out8[4] = c.lowrank_edge;
  out8[5] = c.lowrank_face;
  out8[6] = c.coverage_area;
  out8[7] = c.n_squared;
}

// Direct O(N^2) sum in original order (tests/oracles.cpp:18-33 restated:
// the oracles TU is not linked into the library).
int h3dref_dense_matvec(const double* xyz, std::int64_t n, int kernel_id, double diag,
                        const double* x, double* b) {
  return guarded([&] {
    const PointSet ps = pointset_of(xyz, n);
    const KernelSpec k = kernel_of(kernel_id, diag);
#pragma omp parallel for schedule(dynamic, 64)
    for (std::int64_t i = 0; i < n; ++i) {
      double acc = 0.0;
      for (std::int64_t j = 0; j < n; ++j) {
        if (i == j) continue;
        acc += eval_pair(k, ps.points[static_cast<std::size_t>(i)],
                         ps.points[static_cast<std::size_t>(j)]) * x[j];
      }
      b[i] = acc + k.diagonal * x[i];
    }
  });
}

// Solver (solver.hpp): the IE manufactured-solution experiment and the cell
// constant, for the device GMRES parity tests.
double h3dref_cell_self_integral(double h) { return cell_self_integral(h); }

int h3dref_ie_experiment(int grid_n, double eps, int n_max, std::uint64_t seed, double tol, int restart,
                         int max_iter, int* iterations, int* converged, double* forward_error) {
  return guarded([&] {
    HmatOptions base;
    base.n_max = n_max;
    GmresOptions g;
    g.tol = tol;
    g.restart = restart;
    g.max_iter = max_iter;
    const IeReport r =
        ie_experiment(grid_n, make_kernel(KernelId::Laplace3d), eps, Variant::Hodlr3d, seed, base, g);
    *iterations = r.iterations;
    *converged = r.converged ? 1 : 0;
    *forward_error = r.forward_error;
  });
}

}  // extern "C"
