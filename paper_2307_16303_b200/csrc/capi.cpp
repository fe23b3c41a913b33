// extern "C" boundary (include/h3d_b200.h): exceptions -> status codes.
#include <cstring>
#include <new>
#include <random>
#include <string>

#include <nccl.h>

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
  } catch (const h3db::InvalidArgument& e) {
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
    const ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) throw h3db::NcclFailure(ncclGetErrorString(r));
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
