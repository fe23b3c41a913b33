// extern "C" boundary (include/h3d_b200.h): exceptions -> status codes.
#include <cstring>
#include <new>
#include <random>
#include <string>

#include "nccl_dyn.h"

#include "../../include/h3d_b200.h"
#include "engine.h"

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return H3D_OK;
  } catch (const h3db::DegenerateGeometry& e) {
    g_err = e.what();
    return H3D_EDEGEN_GEOM;
  } catch (const h3db::DegenerateDistribution& e) {
    g_err = e.what();
    return H3D_EDEGEN_DIST;
  } catch (const std::invalid_argument& e) {  // incl. h3db::InvalidArgument
    g_err = e.what();
    return H3D_EINVAL;
  } catch (const h3db::NcclFailure& e) {
    g_err = e.what();
    return H3D_ENCCL;
  } catch (const h3db::CudaError& e) {
    g_err = e.what();
    return H3D_ECUDA;
  } catch (const std::bad_alloc& e) {
    g_err = e.what();
    return H3D_ENOMEM;
  } catch (const std::exception& e) {
    g_err = e.what();
    const bool oom = std::strstr(e.what(), "allocation") != nullptr;
    return oom ? H3D_ENOMEM : H3D_ECUDA;
  }
}

h3db::Engine* eng(h3d_dev* d) { return reinterpret_cast<h3db::Engine*>(d); }
const h3db::Engine* eng(const h3d_dev* d) { return reinterpret_cast<const h3db::Engine*>(d); }

}  // namespace

extern "C" {

const char* h3d_last_error(void) { return g_err.c_str(); }

int h3d_abi_version(void) { return H3D_B200_ABI_VERSION; }

void h3d_default_options(h3d_options* o) {
  std::memset(o, 0, sizeof(*o));
  // h3d::HmatOptions defaults (hmatrix.hpp:16-22), Laplace kernel with K(0)=0
  o->kernel_id = H3D_LAPLACE3D;
  o->diagonal = 0.0;
  o->n_max = 216;
  o->epsilon = 1e-7;
  o->depth_cap = 12;
  o->max_rank = 0;
  o->near_mode = H3D_NEAR_MATRIX_FREE;
  o->device = 0;
  o->shard_rank = 0;
  o->shard_world = 1;
  o->mode_policy = 1;  // auto: direct leaf level, stream/proxy split by the cost model
  o->gather_b = 0;
}

// generate_points(UniformRandom, n, seed) (kernel.cpp:88-95) with the same
// engine and the same top-53-bit mapping (kernel.hpp:24-26).
int h3d_generate_points(int64_t n, uint64_t seed, double* xyz) {
  if (n < 1) {
    g_err = "generate_points: N must be >= 1";
    return H3D_EINVAL;
  }
  std::mt19937_64 gen(seed);
  auto u = [&] { return static_cast<double>(gen() >> 11) * 0x1.0p-53; };
  for (int64_t i = 0; i < n; ++i) {
    const double x = 2.0 * u() - 1.0;
    const double y = 2.0 * u() - 1.0;
    const double z = 2.0 * u() - 1.0;
    xyz[3 * i] = x;
    xyz[3 * i + 1] = y;
    xyz[3 * i + 2] = z;
  }
  return H3D_OK;
}

void h3d_random_vector(int64_t n, uint64_t seed, double* out) {
  std::mt19937_64 gen(seed);
  for (int64_t i = 0; i < n; ++i)
    out[i] = 2.0 * (static_cast<double>(gen() >> 11) * 0x1.0p-53) - 1.0;
}

int h3d_dev_create(const double* xyz, int64_t n, const h3d_options* opt, h3d_dev** out) {
  *out = nullptr;
  return guarded([&] {
    h3d_options o;
    if (opt) o = *opt;
    else h3d_default_options(&o);
    auto* e = new h3db::Engine(xyz, n, o);
    *out = reinterpret_cast<h3d_dev*>(e);
  });
}

void h3d_dev_destroy(h3d_dev* dev) { delete eng(dev); }

int h3d_dev_matvec(h3d_dev* dev, const double* x, double* b, int where, h3d_timing* timing) {
  return guarded([&] {
    if (!dev) throw h3db::InvalidArgument("matvec: null handle");
    std::lock_guard<std::mutex> lk(eng(dev)->mu);
    eng(dev)->matvec(x, b, where == 0, timing);
  });
}

int h3d_dev_matvec_async(h3d_dev* dev, const double* x_dev, double* b_dev, void* stream) {
  return guarded([&] {
    if (!dev) throw h3db::InvalidArgument("matvec: null handle");
    std::lock_guard<std::mutex> lk(eng(dev)->mu);
    eng(dev)->matvec_async(x_dev, b_dev, static_cast<cudaStream_t>(stream));
  });
}

int h3d_dev_profile(h3d_dev* dev, int enable, int64_t capacity) {
  return guarded([&] {
    std::lock_guard<std::mutex> lk(eng(dev)->mu);
    eng(dev)->profile(enable, capacity);
  });
}

int h3d_dev_profile_read(h3d_dev* dev, h3d_timing* sum, int64_t* steps) {
  return guarded([&] {
    std::lock_guard<std::mutex> lk(eng(dev)->mu);
    eng(dev)->profile_read(sum, steps);
  });
}

int h3d_dev_profile_kernels(const h3d_dev* dev, double* ms_sum, int64_t* launches, double* start_sum,
                            int count) {
  return guarded([&] {
    if (!dev || !ms_sum || !launches) throw h3db::InvalidArgument("profile_kernels: null argument");
    eng(dev)->profile_kernels(ms_sum, launches, start_sum, count);
  });
}

int h3d_dev_gmres(h3d_dev* dev, const double* rhs, double* x, int where, double alpha, double beta,
                  double tol, int restart, int max_iter, double* hist, int hist_cap, h3d_gmres_info* info) {
  return guarded([&] {
    if (!dev || !rhs || !x) throw h3db::InvalidArgument("gmres: null argument");
    std::lock_guard<std::mutex> lk(eng(dev)->mu);
    eng(dev)->gmres(rhs, x, where == 0, alpha, beta, tol, restart, max_iter, hist, hist_cap, info);
  });
}

int h3d_dev_direct_matvec(h3d_dev* dev, const double* x, double* b, int where) {
  return guarded([&] {
    if (!dev || !x || !b) throw h3db::InvalidArgument("direct_matvec: null argument");
    std::lock_guard<std::mutex> lk(eng(dev)->mu);
    eng(dev)->direct_matvec(x, b, where == 0);
  });
}

int h3d_dev_comm_ledger(const h3d_dev* dev, h3d_comm_ledger* out) {
  return guarded([&] {
    if (!dev || !out) throw h3db::InvalidArgument("comm_ledger: null argument");
    eng(dev)->comm_ledger(out);
  });
}

int h3d_dev_reference_error(h3d_dev* dev, const double* x, const double* b, int where, int64_t exact_limit,
                            int64_t sample_rows, uint64_t seed, double* out) {
  return guarded([&] {
    if (!dev || !x || !b || !out) throw h3db::InvalidArgument("reference_error: null argument");
    std::lock_guard<std::mutex> lk(eng(dev)->mu);
    *out = eng(dev)->reference_error(x, b, where == 0, exact_limit, sample_rows, seed);
  });
}

int h3d_generate_grid_points(int64_t n, double* xyz) {
  return guarded([&] {
    if (n < 1) throw h3db::InvalidArgument("generate_points: N must be >= 1");
    h3db::tensor_grid_points(n, xyz);
  });
}

double h3d_cell_self_integral(double h) { return h3db::cell_self_integral(h); }

int h3d_dev_stats(const h3d_dev* dev, h3d_stats* out) {
  return guarded([&] { eng(dev)->stats(out); });
}

int h3d_dev_export_tree(const h3d_dev* dev, int32_t* perm, int level, int64_t* offsets) {
  return guarded([&] { eng(dev)->export_tree(perm, level, offsets); });
}

int h3d_dev_export_list(const h3d_dev* dev, int level, int kind, int32_t* offsets, int32_t* ids,
                        int64_t* count) {
  return guarded([&] { *count = eng(dev)->export_list(level, kind, offsets, ids); });
}

int h3d_dev_export_pairs(const h3d_dev* dev, int level, int32_t* x, int32_t* y, int32_t* rank,
                         int64_t* count) {
  return guarded([&] { *count = eng(dev)->export_pairs(level, x, y, rank); });
}

int h3d_nccl_get_id(void* id128) {
  return guarded([&] {
    ncclUniqueId id;
    const ncclResult_t r = h3db::nccl().GetUniqueId(&id);
    if (r != ncclSuccess) throw h3db::NcclFailure(h3db::nccl().GetErrorString(r));
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(id128, &id, sizeof(id));
  });
}

int h3d_dev_attach_nccl(h3d_dev* dev, const void* id128, int rank, int world) {
  return guarded([&] {
    std::lock_guard<std::mutex> lk(eng(dev)->mu);
    eng(dev)->attach_nccl(id128, rank, world);
  });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Host planner (no GPU needed): the shard / layout / work-item logic of the
// engine, exposed so it can be verified on CPU (tests/test_shard_plan.py).
namespace {

h3db::Planner* plan_of(h3d_plan* p) { return reinterpret_cast<h3db::Planner*>(p); }
const h3db::Planner* plan_of(const h3d_plan* p) { return reinterpret_cast<const h3db::Planner*>(p); }

template <class T>
void put(const std::vector<T>& v, void* out, int64_t* count) {
  *count = static_cast<int64_t>(v.size());
  if (out && !v.empty()) std::memcpy(out, v.data(), v.size() * sizeof(T));
}

}  // namespace

extern "C" {

int h3d_plan_create(int depth, int64_t n, const int64_t* offsets, const int32_t* list_off,
                    const int32_t* list_ids, const int64_t* list_counts, int shard_rank,
                    int shard_world, const int* modes, h3d_plan** out) {
  *out = nullptr;
  return guarded([&] {
    if (depth < 0 || depth > 8) throw h3db::InvalidArgument("plan: depth out of range");
    std::vector<std::vector<int64_t>> off(depth + 1);
    std::vector<h3db::LevelLists> lists(depth + 1);
    int64_t po = 0, lo = 0, li = 0;
    for (int l = 0; l <= depth; ++l) {
      const int64_t cnt = 1LL << (3 * l);
      off[l].assign(offsets + po, offsets + po + cnt + 1);
      po += cnt + 1;
      for (int k = 0; k < h3db::kListKinds; ++k) {
        if (l == 0) {
          lists[0].off[k].assign(2, 0);
          continue;
        }
        lists[l].off[k].assign(list_off + lo, list_off + lo + cnt + 1);
        lo += cnt + 1;
        const int64_t c = list_counts[h3db::kListKinds * l + k];
        lists[l].ids[k].assign(list_ids + li, list_ids + li + c);
        li += c;
      }
    }
    std::vector<int> m(modes ? modes : nullptr, modes ? modes + depth + 1 : nullptr);
    auto* p = new h3db::Planner(depth, n, std::move(off), std::move(lists), shard_rank,
                                shard_world, std::move(m));
    *out = reinterpret_cast<h3d_plan*>(p);
  });
}

void h3d_plan_destroy(h3d_plan* p) { delete plan_of(p); }

int h3d_plan_pairs(const h3d_plan* p, int level, int32_t* x, int32_t* y, int64_t* count) {
  return guarded([&] {
    const auto& P = plan_of(p)->pairs(level);
    put(P.X, x, count);
    put(P.Y, y, count);
  });
}

int h3d_plan_set_ranks(h3d_plan* p, int level, const int32_t* ranks) {
  return guarded([&] {
    auto& P = plan_of(p)->pairs(level);
    P.rank.assign(ranks, ranks + P.X.size());
  });
}

int h3d_plan_set_mode(h3d_plan* p, int level, int mode) {
  return guarded([&] { plan_of(p)->set_mode(level, mode); });
}

int h3d_plan_layout(h3d_plan* p) {
  return guarded([&] { plan_of(p)->layout(); });
}

int h3d_plan_array(const h3d_plan* p, const char* name, int level, void* out, int64_t* count) {
  return guarded([&] {
    const h3db::Planner& P = *plan_of(p);
    const std::string nm(name);
    if (nm == "woff") put(P.woff, out, count);
    else if (nm == "soff") put(P.soff, out, count);
    else if (nm == "rowbeg") put(P.rowbeg, out, count);
    else if (nm == "rpad") put(P.rpad, out, count);
    else if (nm == "rows") put(P.rows, out, count);
    else if (nm == "spos") put(P.spos, out, count);
    else if (nm == "pair_wx") put(P.pair_wx.at(level), out, count);
    else if (nm == "pair_wy") put(P.pair_wy.at(level), out, count);
    else if (nm == "pair_rx") put(P.pair_rx.at(level), out, count);
    else if (nm == "pair_ry") put(P.pair_ry.at(level), out, count);
    else if (nm == "pair_cx") put(P.pair_cx.at(level), out, count);
    else if (nm == "pair_cy") put(P.pair_cy.at(level), out, count);
    else if (nm == "p2_items") put(P.p2_items, out, count);
    else if (nm == "p2s_items") put(P.p2s_items, out, count);
    else if (nm == "h2_items") put(P.h2_items, out, count);
    else if (nm == "sym_off") put(P.sym_off, out, count);
    else if (nm == "sym_ids") put(P.sym_ids, out, count);
    else if (nm == "sym_cnt") put(P.sym_cnt, out, count);
    else if (nm == "out_off") put(P.out_off, out, count);
    else if (nm == "in_off") put(P.in_off, out, count);
    else if (nm == "in_pos") put(P.in_pos, out, count);
    else if (nm == "pair_descs") put(P.pair_descs, out, count);
    else if (nm == "pd_level") put(P.pd_level, out, count);
    else if (nm == "fused_descs") put(P.fused_descs, out, count);
    else if (nm == "fd_level") put(P.fd_level, out, count);
    else if (nm == "pg_level") put(P.pg_level, out, count);
    else if (nm == "pc_off") put(P.pc_off, out, count);
    else if (nm == "pc_pos") put(P.pc_pos, out, count);
    else if (nm == "pg_items") put(P.pg_items, out, count);
    else if (nm == "pair_piv") put(P.pair_piv.at(level), out, count);
    else if (nm == "pair_lu") put(P.pair_lu.at(level), out, count);
    else if (nm == "proxy_segs") put(P.proxy_segs, out, count);
    else if (nm == "items") put(P.items, out, count);
    else if (nm == "reds") put(P.reds, out, count);
    else if (nm == "near_off") put(P.near_off, out, count);
    else if (nm == "near_ids") put(P.near_ids, out, count);
    else if (nm == "near_dense") put(P.near_dense, out, count);
    else if (nm == "node_base") put(P.node_base(), out, count);
    else if (nm == "vbase") put(P.vbase, out, count);
    else if (nm == "modes") put(P.modes(), out, count);
    else if (nm == "ranges") {
      const std::vector<int64_t> r{P.leaf0, P.leaf1, P.row0, P.row1};
      put(r, out, count);
    } else if (nm == "rank_rows") {
      std::vector<int64_t> r;
      for (std::size_t i = 0; i < P.rank_row0.size(); ++i) {
        r.push_back(P.rank_row0[i]);
        r.push_back(P.rank_row1[i]);
      }
      put(r, out, count);
    } else if (nm == "sizes") {
      const auto& Z = P.sizes;
      const std::vector<int64_t> r{Z.w_doubles, Z.s_doubles, Z.p_doubles, Z.piv_total,
                                   Z.lu_total, Z.factor_doubles, Z.proxy_units, Z.direct_evals,
                                   Z.sum_rank, Z.npairs, Z.nblocks_ordered, Z.near_blocks,
                                   Z.near_entries};
      put(r, out, count);
    } else {
      throw h3db::InvalidArgument("plan: unknown array " + nm);
    }
  });
}

}  // extern "C"
