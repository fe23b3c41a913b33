// Host orchestration: build (tree -> lists -> plan -> ACA rank pass -> mode
// choice -> layout -> ACA write pass -> proxies) and the matvec launch
// sequence (gather / x all-gather -> phase 1 -> proxy solves -> phase 2).
//
// Reference mapping:
//   Engine::Engine      <- h3d::initialize (hmatrix.cpp:52-151)
//   Engine::enqueue     <- h3d::matvec (hmatrix.cpp:153-226); with shard_world > 1
//                          <- h3d::parallel_matvec (parallel.cpp:111-306)
//   Engine::stats       <- h3d::stats (hmatrix.cpp:228-251)
#include <cstdio>

#include <exception>
#include <thread>

#include "engine.h"
#include "common.cuh"

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <random>
#include <cmath>

#include "nccl_dyn.h"

namespace h3db {

namespace {

using Clock = std::chrono::steady_clock;
double ms_since(Clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}

constexpr int kMaxDepth = 8;       // 8^8 leaves; beyond that the device tables explode
constexpr int kMaxProxyRank = 320; // proxy_solve_kernel's per-warp shared buffer

// Cost model (calibrated on the r01 C3 runs): the
// stream levels are HBM-bound (factor bytes twice per matvec at the bulk-copy
// kernels' measured rate), the proxy levels and the near/direct pass are
// FP64-bound (measured evaluation rates of the regenerating kernels); the two
// lanes overlap imperfectly: T = max(H, D) + kOverlapLoss * min(H, D).
constexpr double kStreamBW = 7.0e12;   // B/s, tile-pipeline read rate
constexpr double kOverlapLoss = 0.35;
constexpr double kStreamPower = 0.0;  // 1/s: power-cap slowdown ~ H^2 (model studies only)
constexpr double kHalfStreamBytes = 8e9;  // B per phase: stream levels at least this large go half
double proxy_rate(int kernel) {  // evaluations / s, Newton-form proxy kernels
  switch (kernel) {
    case kLaplace: return 1.4e12;
    case kR4: return 1.0e12;
    default: return 0.2e12;
  }
}
double near_rate(int kernel) {   // entries / s, near field + direct blocks (each owned
  switch (kernel) {              // pair evaluated once: ~2x the per-entry rate)
    case kLaplace: return 1.9e12;
    case kR4: return 1.4e12;
    default: return 0.25e12;
  }
}

#define NCCL_CHECK(expr)                                                        \
  do {                                                                          \
    ncclResult_t r_ = (expr);                                                   \
    if (r_ != ncclSuccess)                                                      \
      throw NcclFailure(std::string("NCCL error: ") + nccl().GetErrorString(r_) + \
                        " (" #expr ")");                                        \
  } while (0)

}  // namespace

template <class T>
void DevBuf<T>::alloc(std::size_t n) {
  reset();
  if (n == 0) n = 1;
  const cudaError_t e = cudaMalloc(&p_, n * sizeof(T));
  if (e != cudaSuccess) {
    p_ = nullptr;
    (void)cudaGetLastError();
    throw std::runtime_error("device allocation of " + std::to_string(n * sizeof(T)) +
                             " bytes failed: " + cudaGetErrorString(e));
  }
  n_ = n;
}

template <class T>
void DevBuf<T>::reset() {
  if (p_) cudaFree(p_);
  p_ = nullptr;
  n_ = 0;
}

template <class T>
void DevBuf<T>::upload(const T* h, std::size_t n, cudaStream_t s) {
  alloc(n);
  if (n) H3D_CUDA_CHECK(cudaMemcpyAsync(p_, h, n * sizeof(T), cudaMemcpyHostToDevice, s));
}

template class DevBuf<double>;
template class DevBuf<std::int32_t>;
template class DevBuf<std::int64_t>;
template class DevBuf<unsigned>;
template class DevBuf<unsigned long long>;
template class DevBuf<P1Item>;
template class DevBuf<P1Reduce>;
template class DevBuf<ProxySeg>;
template class DevBuf<P2Item>;
template class DevBuf<StreamDesc>;
template class DevBuf<PairDesc>;

Engine::Engine(const double* xyz, std::int64_t n, const h3d_options& opt) : opt_(opt), n_(n) {
  const auto t0 = Clock::now();
  // argument checks in the reference's order (hmatrix.cpp:54-55, octree.cpp:78-82)
  if (n <= 0) throw InvalidArgument("initialize: empty point set");
  if (!(opt.epsilon > 0)) throw InvalidArgument("initialize: eps <= 0");
  if (opt.kernel_id < 0 || opt.kernel_id > 2)
    throw InvalidArgument("initialize: unsupported kernel id (custom kernels cannot cross the C-ABI)");
  if (opt.n_max < 1) throw InvalidArgument("build_tree: n_max must be >= 1");
  if (opt.depth_cap < 0 || opt.depth_cap > 20)
    throw InvalidArgument("build_tree: unreasonable depth cap");
  if (n > 0x7fffffffLL) throw InvalidArgument("initialize: N exceeds int32 point indices");
  if (opt.mode_policy < 0 || opt.mode_policy > 2)
    throw InvalidArgument("initialize: mode_policy must be 0, 1 or 2");
  if (opt.variant < kVariantHodlr3d || opt.variant > kVariantHStrong)
    throw InvalidArgument("unknown variant (0 hodlr3d, 1 hodlr, 2 hstrong)");
  world_ = opt.shard_world < 1 ? 1 : opt.shard_world;
  rank_ = opt.shard_rank;
  if (!(world_ == 1 || world_ == 2 || world_ == 4 || world_ == 8))
    throw InvalidArgument("initialize: shard_world must be 1, 2, 4 or 8 (Morton-subtree ownership)");
  if (rank_ < 0 || rank_ >= world_) throw InvalidArgument("initialize: shard_rank out of range");

  H3D_CUDA_CHECK(cudaSetDevice(opt.device));
  cudaDeviceProp prop{};
  H3D_CUDA_CHECK(cudaGetDeviceProperties(&prop, opt.device));
  sms_ = prop.multiProcessorCount;
  if (const char* t = std::getenv("H3D_TUNE")) {
    const std::string spec(t);
    std::size_t pos = 0;
    while (pos < spec.size()) {
      std::size_t end = spec.find(',', pos);
      if (end == std::string::npos) end = spec.size();
      const std::string kv = spec.substr(pos, end - pos);
      const std::size_t eq = kv.find('=');
      if (eq != std::string::npos) {
        const std::string k = kv.substr(0, eq);
        const int v = std::atoi(kv.c_str() + eq + 1);
        if (k == "p1s") tune_.p1s = v;
        else if (k == "p1p") tune_.p1p = v;
        else if (k == "p2c") tune_.p2c = v;
        else if (k == "p2s") tune_.p2s = v;
        else if (k == "p2p") tune_.p2p = v;
#ifdef H3D_DEVTOOLS
        else if (k == "skip") tune_.skip = v;
        else if (k == "h2w") tune_.h2w = v;
#endif
        else if (k == "nf") tune_.nf = v;
        else if (k == "nfc") tune_.nfc = v;
        else if (k == "fw") tune_.fw = v;
        else if (k == "sol") tune_.sol = v;
        else if (k == "p2o") tune_.p2o = v;
        else if (k == "pps") tune_.pps = v;
        else if (k == "graphs") tune_.graphs = v;
        else if (k == "acab") tune_.acab = v;
        else if (k == "half_search") tune_.half_search = v;
        else if (k == "nfd") tune_.nfd = v;
        else if (k.size() > 4 && k.compare(0, 4, "acat") == 0) {
          const int lv = std::atoi(k.c_str() + 4);
          if (lv > 0 && lv < 16 && (v == 32 || v == 128 || v == 256 || v == 512)) tune_.acat[lv] = v;
        }
      }
      pos = end + 1;
    }
  }
  H3D_CUDA_CHECK(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
  {
    int least = 0, greatest = 0;
    H3D_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    H3D_CUDA_CHECK(cudaStreamCreateWithPriority(&stream2_, cudaStreamNonBlocking, greatest));
    H3D_CUDA_CHECK(cudaStreamCreateWithPriority(&stream4_, cudaStreamNonBlocking, greatest));
    H3D_CUDA_CHECK(cudaStreamCreateWithPriority(&stream3_, cudaStreamNonBlocking, greatest));
  }
  for (auto& e : ev_) H3D_CUDA_CHECK(cudaEventCreate(&e));
  H3D_CUDA_CHECK(cudaEventCreateWithFlags(&done_ev_, cudaEventDisableTiming));
  H3D_CUDA_CHECK(cudaEventCreateWithFlags(&h2_done_, cudaEventDisableTiming));
  for (int k = 0; k < 3; ++k) {
    H3D_CUDA_CHECK(cudaEventCreateWithFlags(&fork_[k], cudaEventDisableTiming));
    H3D_CUDA_CHECK(cudaEventCreateWithFlags(&join_[k], cudaEventDisableTiming));
  }

  auto t = Clock::now();
  build_tree(xyz);
  ms_tree_ = ms_since(t);
  t = Clock::now();
  build_lists();
  ms_lists_ = ms_since(t);

  // initial modes: direct leaf level (auto: small leaves are cheaper to
  // evaluate than to compress), stream/proxy for the rest decided after ranks
  modes_.assign(L_ + 1, kModeStream);
  if (opt_.mode_policy == 1 && L_ >= 1 && opt_.n_max <= 128) modes_[L_] = kModeDirect;
  if (opt_.mode_policy == 2) {
    for (int l = 1; l <= L_ && l < 16; ++l) {
      const int m = opt_.level_modes[l];
      if (m < 0 || m > kModeLast)
        throw InvalidArgument("initialize: level_modes entries must be 0, 1, 2, 3, 4, 5 or 6");
      if (m == kModeDirect && l != L_)
        throw InvalidArgument("initialize: direct mode is only valid at the leaf level");
      modes_[l] = m;
    }
  }
  plan_ = std::make_unique<Planner>(L_, n_, off_, lists_, rank_, world_, modes_);
  // stored near field: the dense leaf blocks in cached mode (the reference's
  // DenseMode::Cached); the direct leaf-level blocks with H3D_TUNE nfd=1
  plan_->set_near_storage((opt_.near_mode == H3D_NEAR_STORED ? 1 : 0) | (tune_.nfd ? 2 : 0));
  // the rank-independent part of the layout (leaf plan, near-field lists) on
  // a host thread while the ACA rank pass runs on the device
  std::exception_ptr leaf_err;
  std::thread leaf_thread([this, &leaf_err] {
    try {
      plan_->layout_leaf();
    } catch (...) {
      leaf_err = std::current_exception();
    }
  });
  t = Clock::now();
  try {
    run_aca(false);
  } catch (...) {
    leaf_thread.join();
    throw;
  }
  ms_aca_rank_ = ms_since(t);
  t = Clock::now();
  leaf_thread.join();
  if (leaf_err) std::rethrow_exception(leaf_err);
  choose_modes();
  plan_->layout();
  upload_plan();
  ms_plan_ = ms_since(t);
  t = Clock::now();
  single_pass_ = finish_single_pass();
  if (!single_pass_) {
    for (int l = 1; l <= L_; ++l)
      if (plan_->mode(l) == kModeHalf)
        throw InvalidArgument("initialize: half mode (5) needs the single-pass build, whose pivot / LU pool "
                              "did not fit in device memory; use stream or proxy mode");
    run_aca(true);
  }
  ms_aca_write_ = ms_since(t);
  t = Clock::now();
  if (n_segs_all_ > 0) {
    launch_proxy_gather(segs_all_.get(), n_segs_all_, piv_.get(), px_.get(), py_.get(), pz_.get(),
                        center_.get(), q4_.get(), q4c_.get(), stream_);
    int max_r = 0;
    for (const auto& sg : plan_->proxy_segs) max_r = std::max(max_r, sg.r);
    launch_lu_invert(segs_all_.get(), n_segs_all_, lu_.get(), lu_total_, max_r, stream_);
  }
  if (!plan_->fused_descs.empty()) {
    // triangular inverses of the fused pairs' pivot LUs (one side-0 segment each)
    std::vector<ProxySeg> segs;
    int max_r = 0;
    for (const auto& d : plan_->fused_descs) {
      ProxySeg sg{};
      sg.lu_off = d.lu_off;
      sg.piv_off = d.piv_off;
      sg.r = d.r;
      sg.side = 0;
      segs.push_back(sg);
      max_r = std::max(max_r, d.r);
    }
    DevBuf<ProxySeg> d_segs;
    d_segs.upload(segs, stream_);
    launch_lu_invert(d_segs.get(), static_cast<std::int64_t>(segs.size()), lu_.get(), lu_total_, max_r,
                     stream_);
    H3D_CUDA_CHECK(cudaStreamSynchronize(stream_));
  }
  H3D_CUDA_CHECK(cudaStreamSynchronize(stream_));
  ms_post_ = ms_since(t);
  t = Clock::now();
  near_scan();
  H3D_CUDA_CHECK(cudaStreamSynchronize(stream_));
  ms_near_ = ms_since(t);
  ms_total_ = ms_since(t0);
}

Engine::~Engine() {
  for (auto& g : graphs_)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  for (auto e : prof_ev_)
    if (e) cudaEventDestroy(e);
  if (nccl_comm_) nccl().CommDestroy(static_cast<ncclComm_t>(nccl_comm_));
  for (auto& e : ev_)
    if (e) cudaEventDestroy(e);
  if (done_ev_) cudaEventDestroy(done_ev_);
  if (h2_done_) cudaEventDestroy(h2_done_);
  for (int k = 0; k < 3; ++k) {
    if (fork_[k]) cudaEventDestroy(fork_[k]);
    if (join_[k]) cudaEventDestroy(join_[k]);
  }
  if (stream4_) cudaStreamDestroy(stream4_);
  if (stream3_) cudaStreamDestroy(stream3_);
  if (stream2_) cudaStreamDestroy(stream2_);
  if (stream_) cudaStreamDestroy(stream_);
}

void Engine::check_flags(const char* where) {
  unsigned f = 0;
  H3D_CUDA_CHECK(cudaMemcpyAsync(&f, flags_.get(), sizeof(unsigned), cudaMemcpyDeviceToHost, stream_));
  H3D_CUDA_CHECK(cudaStreamSynchronize(stream_));
  if (f & kFlagOutOfDomain) throw InvalidArgument("build_tree: point outside the domain cube");
  if (f & kFlagDegenGeom)
    throw DegenerateGeometry(std::string("coincident distinct points in block (") + where + ")");
}

// ---------------------------------------------------------------- tree
void Engine::build_tree(const double* xyz) {
  const int cap = opt_.depth_cap;
  DevBuf<double> xyz_d;
  xyz_d.upload(xyz, static_cast<std::size_t>(3 * n_), stream_);
  flags_.alloc(1);
  H3D_CUDA_CHECK(cudaMemsetAsync(flags_.get(), 0, sizeof(unsigned), stream_));
  DevBuf<unsigned long long> codes, codes_s;
  DevBuf<std::int32_t> idx;
  codes.alloc(n_);
  codes_s.alloc(n_);
  idx.alloc(n_);
  perm_.alloc(n_);
  launch_morton_codes(xyz_d.get(), n_, cap, codes.get(), idx.get(), flags_.get(), stream_);
  check_flags("build_tree");
  const int end_bit = 3 * cap;
  if (end_bit > 0) {
    const std::size_t tb = radix_sort_temp_bytes(n_, end_bit);
    DevBuf<unsigned char> tmp;
    tmp.alloc(tb);
    radix_sort_pairs(tmp.get(), tb, codes.get(), codes_s.get(), idx.get(), perm_.get(), n_, end_bit,
                     stream_);
    H3D_CUDA_CHECK(cudaStreamSynchronize(stream_));
  } else {
    H3D_CUDA_CHECK(cudaMemcpyAsync(codes_s.get(), codes.get(), n_ * 8, cudaMemcpyDeviceToDevice, stream_));
    H3D_CUDA_CHECK(cudaMemcpyAsync(perm_.get(), idx.get(), n_ * 4, cudaMemcpyDeviceToDevice, stream_));
  }
  codes.reset();
  idx.reset();
  // depth = min l with max occupancy < n_max (octree.cpp:110-136)
  DevBuf<unsigned long long> maxocc;
  maxocc.alloc(cap + 1);
  H3D_CUDA_CHECK(cudaMemsetAsync(maxocc.get(), 0, (cap + 1) * 8, stream_));
  launch_depth_scan(codes_s.get(), n_, cap, maxocc.get(), stream_);
  std::vector<unsigned long long> occ(cap + 1);
  H3D_CUDA_CHECK(cudaMemcpyAsync(occ.data(), maxocc.get(), (cap + 1) * 8, cudaMemcpyDeviceToHost, stream_));
  H3D_CUDA_CHECK(cudaStreamSynchronize(stream_));
  int depth = -1;
  for (int l = 0; l <= cap; ++l)
    if (occ[l] < static_cast<unsigned long long>(opt_.n_max)) {
      depth = l;
      break;
    }
  if (depth < 0)
    throw DegenerateDistribution("build_tree: depth cap " + std::to_string(cap) +
                                 " exceeded; distribution too concentrated for n_max = " +
                                 std::to_string(opt_.n_max));
  if (depth > kMaxDepth)
    throw InvalidArgument("initialize: tree depth " + std::to_string(depth) +
                          " exceeds the device engine's limit of " + std::to_string(kMaxDepth));
  L_ = depth;
  off_.resize(L_ + 1);
  for (int l = 0; l <= L_; ++l) {
    const std::int64_t cnt = 1LL << (3 * l);
    DevBuf<std::int64_t> o;
    o.alloc(cnt + 1);
    launch_node_offsets(codes_s.get(), n_, cap, l, o.get(), stream_);
    off_[l].resize(cnt + 1);
    H3D_CUDA_CHECK(cudaMemcpyAsync(off_[l].data(), o.get(), (cnt + 1) * 8, cudaMemcpyDeviceToHost, stream_));
    H3D_CUDA_CHECK(cudaStreamSynchronize(stream_));
  }
  perm_h_.resize(n_);
  H3D_CUDA_CHECK(cudaMemcpyAsync(perm_h_.data(), perm_.get(), n_ * 4, cudaMemcpyDeviceToHost, stream_));
  px_.alloc(n_);
  py_.alloc(n_);
  pz_.alloc(n_);
  launch_permute_points(xyz_d.get(), perm_.get(), n_, px_.get(), py_.get(), pz_.get(), stream_);
  p4_.alloc(4 * n_);
  launch_pack_points(px_.get(), py_.get(), pz_.get(), n_, p4_.get(), stream_);
  leaf_off_.upload(off_[L_], stream_);
  H3D_CUDA_CHECK(cudaStreamSynchronize(stream_));
}

// ---------------------------------------------------------------- lists
void Engine::build_lists() {
  lists_.assign(L_ + 1, LevelLists{});
  for (int k = 0; k < kListKinds; ++k) lists_[0].off[k].assign(2, 0);
  if (L_ == 0) return;
  const std::int64_t maxcnt = 1LL << (3 * L_);
  const std::size_t tb = scan_temp_bytes(maxcnt);
  DevBuf<unsigned char> tmp;
  tmp.alloc(tb);
  DevBuf<std::int32_t> counts, offs;
  counts.alloc(kListKinds * (maxcnt + 1));
  offs.alloc(kListKinds * (maxcnt + 1));
  for (int l = 1; l <= L_; ++l) {
    const std::int64_t cnt = 1LL << (3 * l);
    H3D_CUDA_CHECK(cudaMemsetAsync(counts.get(), 0, kListKinds * (cnt + 1) * 4, stream_));
    launch_list_counts(l, opt_.variant, counts.get(), stream_);
    for (int k = 0; k < kListKinds; ++k)
      exclusive_scan_i32(tmp.get(), tb, counts.get() + k * (cnt + 1), offs.get() + k * (cnt + 1), cnt,
                         stream_);
    std::vector<std::int32_t> hoff(kListKinds * (cnt + 1));
    H3D_CUDA_CHECK(cudaMemcpyAsync(hoff.data(), offs.get(), hoff.size() * 4, cudaMemcpyDeviceToHost, stream_));
    H3D_CUDA_CHECK(cudaStreamSynchronize(stream_));
    DevBuf<std::int32_t> ids[kListKinds];
    std::int32_t* idp[kListKinds];
    for (int k = 0; k < kListKinds; ++k) {
      lists_[l].off[k].assign(hoff.begin() + k * (cnt + 1), hoff.begin() + (k + 1) * (cnt + 1));
      ids[k].alloc(lists_[l].off[k][cnt]);
      idp[k] = ids[k].get();
    }
    launch_list_fill(l, opt_.variant, offs.get(), idp, stream_);
    for (int k = 0; k < kListKinds; ++k) {
      lists_[l].ids[k].resize(lists_[l].off[k][cnt]);
      if (!lists_[l].ids[k].empty())
        H3D_CUDA_CHECK(cudaMemcpyAsync(lists_[l].ids[k].data(), ids[k].get(),
                                       lists_[l].ids[k].size() * 4, cudaMemcpyDeviceToHost, stream_));
    }
    H3D_CUDA_CHECK(cudaStreamSynchronize(stream_));
  }
}

// ---------------------------------------------------------------- ACA
void Engine::run_aca(bool write) {
  DevBuf<unsigned long long> counter;
  counter.alloc(1);
  std::size_t free_b = 0, total_b = 0;
  H3D_CUDA_CHECK(cudaMemGetInfo(&free_b, &total_b));
  if (!write) free_mem_ = free_b;
  if (!write && std::getenv("H3D_TWO_PASS") == nullptr) {
    // single-pass build: a bump pool for every pair's pivots + packed LU
    // (sum r^2 + r doubles; C3 ~3.6 GB, C5 ~35 GB), a fifth of free memory
    const std::size_t cap_b = free_b / 5;
    pool_.alloc(std::max<std::size_t>(cap_b / 8, 1));
    pool_ctr_.alloc(1);
    H3D_CUDA_CHECK(cudaMemsetAsync(pool_ctr_.get(), 0, 8, stream_));
    pool_off_.clear();
    pool_off_.resize(static_cast<std::size_t>(L_) + 1);
    pool_ok_ = true;
  }
  for (int l = 1; l <= L_; ++l) {
    auto& P = plan_->pairs(l);
    const std::int64_t np = static_cast<std::int64_t>(P.X.size());
    if (np == 0) continue;
    if (!write && l < 16 && tune_.acat[l] > 0) P.threads = tune_.acat[l];
    const int mode = plan_->mode(l);
    const auto t_level = Clock::now();
    std::vector<std::int64_t> xb(np), yb(np);
    std::vector<std::int32_t> m(np), nn(np);
    for (std::int64_t p = 0; p < np; ++p) {
      xb[p] = off_[l][P.X[p]];
      yb[p] = off_[l][P.Y[p]];
      m[p] = static_cast<std::int32_t>(node_size(l, P.X[p]));
      nn[p] = static_cast<std::int32_t>(node_size(l, P.Y[p]));
    }
    DevBuf<std::int64_t> d_xb, d_yb, d_wx, d_wy, d_po, d_lo;
    DevBuf<std::int32_t> d_m, d_n, d_rank, d_rx, d_ry, d_cx, d_cy, d_order;
    {
      std::vector<std::int32_t> order;
      order.reserve(static_cast<std::size_t>(np));
      // claim order: touching pairs (the highest ranks, r^2 (m + n) panel
      // traffic each) first, so their long ACAs do not form the level's tail
      for (int pass = 0; pass < 2; ++pass)
        for (std::int64_t p = 0; p < np; ++p)
          if (boxes_touch(P.X[p], P.Y[p]) == (pass == 0)) order.push_back(static_cast<std::int32_t>(p));
      d_order.upload(order, stream_);
    }
    d_xb.upload(xb, stream_);
    d_yb.upload(yb, stream_);
    d_m.upload(m, stream_);
    d_n.upload(nn, stream_);
    d_rank.alloc(np);
    int level_max_rank = 0;
    if (write) {
      for (std::int64_t p = 0; p < np; ++p) level_max_rank = std::max(level_max_rank, P.rank[p]);
      if (mode == kModeStream || mode == kModePair) {
        d_wx.upload(plan_->pair_wx[l], stream_);
        d_wy.upload(plan_->pair_wy[l], stream_);
        d_rx.upload(plan_->pair_rx[l], stream_);
        d_ry.upload(plan_->pair_ry[l], stream_);
        d_cx.upload(plan_->pair_cx[l], stream_);
        d_cy.upload(plan_->pair_cy[l], stream_);
      } else {
        d_po.upload(plan_->pair_piv[l], stream_);
        d_lo.upload(plan_->pair_lu[l], stream_);
      }
    }
    const int ms = (P.max_m + 1) & ~1, ns = (P.max_n + 1) & ~1;
    int cap_ws;
    if (write) {
      cap_ws = std::max(1, level_max_rank);
    } else {
      cap_ws = std::min(P.max_mn, P.threads == 32 ? 128 : 256);
      if (opt_.max_rank > 0) cap_ws = static_cast<int>(std::min<std::int64_t>(cap_ws, opt_.max_rank));
      cap_ws = std::max(cap_ws, 1);
    }
    for (;;) {
      const std::int64_t slot_doubles =
          static_cast<std::int64_t>(cap_ws + 1) * (ms + ns) + (ms + ns + 7) / 8 + 2;
      const std::size_t smem = aca_smem_bytes(P.threads, cap_ws);
      if (smem > 227u * 1024u)
        throw InvalidArgument("initialize: ACA rank at level " + std::to_string(l) + " exceeds " +
                              std::to_string(cap_ws / 2) +
                              " (shared-memory pivot state); raise eps or set max_rank");
      // few huge blocks (top levels): one thread-block cluster per pair so the
      // whole GPU works on them; fixed per level for rank/write determinism
      if (P.cluster == 0) {
        int cl = 1;
        if (P.threads >= 256 && np * 4 <= sms_) {
          cl = 2;
          while (cl < 16 && np * cl * 2 <= sms_) cl <<= 1;
        }
        P.cluster = cl;
      }
      const std::int64_t budget = std::max<std::int64_t>(
          std::min<std::int64_t>(static_cast<std::int64_t>(free_b / 4), 24LL << 30), 256LL << 20);
      AcaArgs a;
      a.npairs = np;
      a.xb = d_xb.get();
      a.m = d_m.get();
      a.yb = d_yb.get();
      a.n = d_n.get();
      a.px = px_.get();
      a.py = py_.get();
      a.pz = pz_.get();
      a.kernel = opt_.kernel_id;
      a.diag = opt_.diagonal;
      a.eps = opt_.epsilon;
      a.max_rank = opt_.max_rank;
      a.slot_doubles = slot_doubles;
      a.cap_ws = cap_ws;
      a.ms = ms;
      a.ns = ns;
      a.rank_out = d_rank.get();
      if (write && (mode == kModeStream || mode == kModePair)) {
        a.row_major = mode == kModePair ? 1 : 0;
        a.W = W_.get();
        a.wx = d_wx.get();
        a.rx = d_rx.get();
        a.wy = d_wy.get();
        a.ry = d_ry.get();
        a.cx = d_cx.get();
        a.cy = d_cy.get();
      }
      if (write && (mode == kModeProxy || mode == kModeFused)) {
        a.piv = piv_.get();
        a.lu = lu_.get();
        a.piv_off = d_po.get();
        a.lu_off = d_lo.get();
      }
      a.flags = flags_.get();
      a.counter = counter.get();
      if (!write && pool_ok_) {
        auto& po = pool_off_[static_cast<std::size_t>(l)];
        if (!po) po = std::make_unique<DevBuf<std::int64_t>>();
        if (po->size() != static_cast<std::size_t>(np)) po->alloc(static_cast<std::size_t>(np));
        a.pool = pool_.get();
        a.pool_ctr = pool_ctr_.get();
        a.pool_cap = static_cast<std::int64_t>(pool_.size());
        a.pool_off = po->get();
      }
      H3D_CUDA_CHECK(cudaMemsetAsync(flags_.get(), 0, 4, stream_));
      // one launch: claims [c0, c0 + nc) of the order, cluster cl
      auto launch_group = [&](std::int64_t c0, std::int64_t nc, int cl) {
        if (nc <= 0) return;
        int bps = cl > 1 ? 1 : aca_blocks_per_sm(P.threads, opt_.kernel_id, smem);
        if (tune_.acab > 0 && cl <= 1) bps = std::min(bps, tune_.acab);
        std::int64_t slots =
            cl > 1 ? std::min<std::int64_t>(nc, std::max(1, aca_max_clusters(P.threads, opt_.kernel_id, cl, smem)))
                   : std::min<std::int64_t>(nc, static_cast<std::int64_t>(bps) * sms_);
        slots = std::min<std::int64_t>(slots, std::max<std::int64_t>(1, budget / (slot_doubles * 8)));
        DevBuf<double> ws;
        ws.alloc(static_cast<std::size_t>(slots * slot_doubles));
        H3D_CUDA_CHECK(cudaMemsetAsync(counter.get(), 0, 8, stream_));
        AcaArgs g = a;
        g.ws = ws.get();
        g.order = d_order.get() + c0;
        g.nclaims = nc;
        if (cl > 1)
          launch_aca_cluster(g, P.threads, cl, static_cast<int>(slots), stream_);
        else
          launch_aca(g, P.threads, static_cast<int>(slots), stream_);
        H3D_CUDA_CHECK(cudaStreamSynchronize(stream_));  // ws is freed on return
      };
      launch_group(0, np, P.cluster);
      unsigned f = 0;
      H3D_CUDA_CHECK(cudaMemcpyAsync(&f, flags_.get(), 4, cudaMemcpyDeviceToHost, stream_));
      H3D_CUDA_CHECK(cudaStreamSynchronize(stream_));
      if (f & kFlagDegenGeom) throw DegenerateGeometry("coincident distinct points in block");
      if (f & kFlagPoolFull) pool_ok_ = false;  // the write pass recomputes the factors instead
      if (f & kFlagAcaOverflow) {
        if (write || cap_ws >= P.max_mn)
          throw std::logic_error("ACA workspace overflow in the write pass");
        cap_ws = std::min(2 * cap_ws, P.max_mn);
        continue;
      }
      break;
    }
    if (l < 16) level_aca_ms_[l] += ms_since(t_level);
    std::vector<std::int32_t> rk(np);
    H3D_CUDA_CHECK(cudaMemcpyAsync(rk.data(), d_rank.get(), np * 4, cudaMemcpyDeviceToHost, stream_));
    H3D_CUDA_CHECK(cudaStreamSynchronize(stream_));
    if (write) {
      if (rk != P.rank) throw std::logic_error("ACA write pass diverged from the rank pass");
    } else {
      P.rank = std::move(rk);
    }
  }
  if (!write && pool_ok_) {
    // keep only the used part of the pool (the planner sizes W from the
    // memory that is free after the rank pass)
    unsigned long long used = 0;
    H3D_CUDA_CHECK(cudaMemcpyAsync(&used, pool_ctr_.get(), 8, cudaMemcpyDeviceToHost, stream_));
    H3D_CUDA_CHECK(cudaStreamSynchronize(stream_));
    DevBuf<double> exact;
    exact.alloc(std::max<std::size_t>(static_cast<std::size_t>(used), 1));
    if (used > 0)
      H3D_CUDA_CHECK(cudaMemcpyAsync(exact.get(), pool_.get(), used * 8, cudaMemcpyDeviceToDevice, stream_));
    H3D_CUDA_CHECK(cudaStreamSynchronize(stream_));
    pool_.swap(exact);
    free_mem_ -= std::min<std::size_t>(free_mem_, static_cast<std::size_t>(used) * 8);
  }
  if (!write && !pool_ok_) {
    pool_.reset();
    pool_off_.clear();
  }
}

// Single-pass build, after the layout: proxy / fused levels take their pivots
// and packed LU from the rank pass's pool (compaction into the planner's
// offsets); stream / pair levels get explicit factors generated from the same
// pivots + LU (triangular inverses, U = K(X, tau) R^-1, V = K(Y, sigma) L^-T)
// instead of a second ACA pass. Returns false when the pool overflowed (the
// caller runs the ACA write pass).
bool Engine::finish_single_pass() {
  if (!pool_ok_) {
    pool_.reset();
    pool_off_.clear();
    return false;
  }
  for (int l = 1; l <= L_; ++l) {
    auto& P = plan_->pairs(l);
    const std::int64_t np = static_cast<std::int64_t>(P.X.size());
    if (np == 0) continue;
    const int mode = plan_->mode(l);
    DevBuf<std::int32_t> d_rank;
    d_rank.upload(P.rank, stream_);
    const std::int64_t* poff = pool_off_[static_cast<std::size_t>(l)]->get();
    if (mode == kModeProxy || mode == kModeFused || two_groups(mode)) {
      DevBuf<std::int64_t> d_po, d_lo;
      d_po.upload(plan_->pair_piv[l], stream_);
      d_lo.upload(plan_->pair_lu[l], stream_);
      launch_aca_compact(pool_.get(), poff, d_rank.get(), np, piv_.get(), d_po.get(),
                         mode == kModeHalf ? nullptr : lu_.get(), d_lo.get(), stream_);
      H3D_CUDA_CHECK(cudaStreamSynchronize(stream_));
      // half levels also get the explicit U' = K(X, tau) R^-1 L^-1 (below)
      if (mode != kModeHalf) continue;
    }
    // stream / pair / half level: pivots + LU into a temporary block array,
    // its triangular inverses, then the explicit factors straight into W - in
    // chunks of pairs whose temporaries stay under ~2 GB (C5 level 5 alone
    // would need ~20 GB beside the pool and W)
    constexpr std::int64_t kChunkDoubles = 128LL << 20;
    for (std::int64_t p0 = 0; p0 < np;) {
      std::int64_t p1 = p0, ptot = 0, ltot = 0;
      int max_r = 0;
      std::vector<std::int64_t> po, lo, xb, yb, wx, wy;
      std::vector<std::int32_t> m, nn, rx, ry, cx, cy;
      std::vector<ProxySeg> segs;
      while (p1 < np && (p1 == p0 || ltot < kChunkDoubles)) {
        const std::int64_t p = p1++;
        const std::int64_t r = P.rank[p];
        po.push_back(ptot);
        lo.push_back(ltot);
        ptot += 2 * r;
        ltot += r * r + (r & 1);
        max_r = std::max<int>(max_r, static_cast<int>(r));
        xb.push_back(off_[l][P.X[p]]);
        yb.push_back(off_[l][P.Y[p]]);
        m.push_back(static_cast<std::int32_t>(node_size(l, P.X[p])));
        nn.push_back(static_cast<std::int32_t>(node_size(l, P.Y[p])));
        wx.push_back(plan_->pair_wx[l][p]);
        wy.push_back(plan_->pair_wy[l][p]);
        rx.push_back(plan_->pair_rx[l][p]);
        ry.push_back(plan_->pair_ry[l][p]);
        cx.push_back(plan_->pair_cx[l][p]);
        cy.push_back(plan_->pair_cy[l][p]);
        ProxySeg sg{};
        sg.lu_off = lo.back();
        sg.piv_off = po.back();
        sg.r = static_cast<std::int32_t>(r);
        sg.side = 0;
        segs.push_back(sg);
      }
      const std::int64_t nc = p1 - p0;
      if (max_r > 0) {
        DevBuf<std::int32_t> tpiv, d_m, d_n;
        DevBuf<double> tlu;
        DevBuf<std::int64_t> d_po, d_lo, d_xb, d_yb, d_wx, d_wy;
        DevBuf<std::int32_t> d_rx, d_ry, d_cx, d_cy;
        DevBuf<ProxySeg> d_segs;
        tpiv.alloc(static_cast<std::size_t>(std::max<std::int64_t>(ptot, 1)));
        tlu.alloc(static_cast<std::size_t>(std::max<std::int64_t>(2 * ltot, 1)));
        d_po.upload(po, stream_);
        d_lo.upload(lo, stream_);
        launch_aca_compact(pool_.get(), poff + p0, d_rank.get() + p0, nc, tpiv.get(), d_po.get(), tlu.get(),
                           d_lo.get(), stream_);
        d_segs.upload(segs, stream_);
        launch_lu_invert(d_segs.get(), nc, tlu.get(), ltot, max_r, stream_);
        d_xb.upload(xb, stream_);
        d_yb.upload(yb, stream_);
        d_m.upload(m, stream_);
        d_n.upload(nn, stream_);
        d_wx.upload(wx, stream_);
        d_wy.upload(wy, stream_);
        d_rx.upload(rx, stream_);
        d_ry.upload(ry, stream_);
        d_cx.upload(cx, stream_);
        d_cy.upload(cy, stream_);
        FactorGenArgs fa;
        fa.npairs = nc;
        fa.xb = d_xb.get();
        fa.m = d_m.get();
        fa.yb = d_yb.get();
        fa.n = d_n.get();
        fa.rank = d_rank.get() + p0;
        fa.piv = tpiv.get();
        fa.piv_off = d_po.get();
        fa.inv = tlu.get();
        fa.inv_total = ltot;
        fa.inv_off = d_lo.get();
        fa.px = px_.get();
        fa.py = py_.get();
        fa.pz = pz_.get();
        fa.kernel = opt_.kernel_id;
        fa.W = W_.get();
        fa.wx = d_wx.get();
        fa.cx = d_cx.get();
        fa.rx = d_rx.get();
        fa.wy = d_wy.get();
        fa.cy = d_cy.get();
        fa.ry = d_ry.get();
        fa.row_major = mode == kModePair ? 1 : 0;
        fa.full = mode == kModeHalf ? 1 : 0;
        fa.max_r = max_r;
        launch_factor_gen(fa, stream_);
        H3D_CUDA_CHECK(cudaStreamSynchronize(stream_));
      }
      p0 = p1;
    }
  }
  pool_.reset();
  pool_off_.clear();
  return true;
}

// ---------------------------------------------------------------- modes
// Auto policy: the FP64 pipes (proxy regeneration, near field, direct leaf
// blocks) and HBM (factor streaming) are separate resources; pick the
// stream/proxy split of the upper levels that minimises
//   max(stream, compute_1) + max(stream, compute_2 + near + direct)
// subject to the factor pool fitting in free memory.
void Engine::choose_modes() {
  if (opt_.mode_policy == 2) {
    for (int l = 1; l <= L_; ++l) {
      if (plan_->mode(l) == kModeHalf && !plan_->pairs(l).X.empty() && opt_.kernel_id != kLaplace &&
          opt_.kernel_id != kR4)
        throw InvalidArgument("initialize: half mode (5) is for the smooth kernels (laplace3d, r4): with "
                              "cos(r)/r the explicit U' = K(X, tau) (LR)^-1 loses accuracy; use proxy or "
                              "stream mode there");
      if (plan_->mode(l) == kModePair) {
        const auto& rk = plan_->pairs(l).rank;
        if (!rk.empty() && *std::max_element(rk.begin(), rk.end()) > kPairMaxRp)
          throw InvalidArgument("initialize: level " + std::to_string(l) + " has ranks above " +
                                std::to_string(kPairMaxRp) + "; use stream mode there");
        continue;
      }
      if (plan_->mode(l) == kModeFused) {
        const auto& P = plan_->pairs(l);
        for (std::size_t p = 0; p < P.X.size(); ++p) {
          if (P.rank[p] > kFusedMaxRank)
            throw InvalidArgument("initialize: level " + std::to_string(l) + " has ranks above " +
                                  std::to_string(kFusedMaxRank) + "; use proxy or stream mode there");
          const std::int64_t m = node_size(l, P.X[p]), n = node_size(l, P.Y[p]);
          if (std::max(m, n) > fused_max_node())
            throw InvalidArgument("initialize: level " + std::to_string(l) +
                                  " has nodes with more points than the fused pass holds (" +
                                  std::to_string(fused_max_node()) + "); use proxy or stream mode there");
        }
        continue;
      }
      if (plan_->mode(l) != kModeProxy && plan_->mode(l) != kModeSplit) continue;
      const auto& rk = plan_->pairs(l).rank;
      if (!rk.empty() && *std::max_element(rk.begin(), rk.end()) > kMaxProxyRank)
        throw InvalidArgument("initialize: level " + std::to_string(l) + " has ranks above " +
                              std::to_string(kMaxProxyRank) + "; use stream mode there");
    }
  }
  if (opt_.mode_policy != 1) return;
  std::vector<int> cand;
  // per level: units (sum r (m + n)), the X-side part (sum r m), sum r^2
  std::vector<double> units(L_ + 1, 0.0), ux(L_ + 1, 0.0), lu(L_ + 1, 0.0);
  std::vector<int> maxr(L_ + 1, 0);
  for (int l = 1; l <= L_; ++l) {
    const auto& P = plan_->pairs(l);
    if (plan_->mode(l) == kModeDirect || P.X.empty()) continue;
    for (std::size_t p = 0; p < P.X.size(); ++p) {
      const double r = P.rank[p];
      units[l] += r * static_cast<double>(node_size(l, P.X[p]) + node_size(l, P.Y[p]));
      ux[l] += r * static_cast<double>(node_size(l, P.X[p]));
      lu[l] += r * r;
      maxr[l] = std::max(maxr[l], P.rank[p]);
    }
    cand.push_back(l);
  }
  // phase-2 compute independent of the split: near field + direct leaf blocks
  double fixed = 0.0;
  {
    const auto& lst = lists_[L_];
    for (std::int64_t x = 0; x < (1LL << (3 * L_)); ++x) {
      const double mx = static_cast<double>(node_size(L_, x));
      if (mx == 0) continue;
      double nsum = mx;
      if (L_ > 0) {
        for (int k = 1; k < kListKinds; ++k)
          for (std::int32_t e = lst.off[k][x]; e < lst.off[k][x + 1]; ++e)
            nsum += static_cast<double>(node_size(L_, lst.ids[k][e]));
        if (plan_->mode(L_) == kModeDirect)
          for (std::int32_t e = lst.off[0][x]; e < lst.off[0][x + 1]; ++e)
            nsum += static_cast<double>(node_size(L_, lst.ids[0][e]));
      }
      fixed += mx * nsum;
    }
    fixed /= static_cast<double>(world_);
  }
  const double budget = 0.8 * static_cast<double>(free_mem_) - 64.0 * static_cast<double>(n_) -
                        (2 << 30);
  const double Rp = proxy_rate(opt_.kernel_id), Rn = near_rate(opt_.kernel_id);
  // half levels (mode 5) form U' = K(X, tau) (LR)^-1 explicitly: fine for the
  // smooth kernels, unstable for the oscillatory cos(r)/r (an ill-conditioned
  // R mixed into every column of U', measured 0.06-0.16 relative error on
  // the Helmholtz goldens), so auto offers it for Laplace and 1/r^4 only,
  // and only when the single-pass pool kept every pair's pivots + LU
  const bool half_ok = (opt_.kernel_id == kLaplace || opt_.kernel_id == kR4) && pool_ok_;
  // the search covers proxy / stream (H3D_TUNE half_search=1: half too, for
  // model studies); half replaces large stream levels afterwards (below)
  const int nopt = half_ok && tune_.half_search ? 3 : 2;  // 0 proxy, 1 stream, 2 half
  const unsigned ncand = static_cast<unsigned>(cand.size());
  unsigned ncomb = 1;
  for (unsigned i = 0; i < ncand; ++i) ncomb *= static_cast<unsigned>(nopt);
  double best = 1e300;
  unsigned best_code = 0;
  const bool dbg = std::getenv("H3D_MODEL_PRINT") != nullptr;
  // stream levels that will become half levels (below) need only U' in W
  auto to_half = [&](int l) { return half_ok && l > 1 && 8.0 * units[l] >= kHalfStreamBytes; };
  for (unsigned code = 0; code < ncomb; ++code) {
    double sbytes = 0.0, evals = 0.0, lub = 0.0, wbytes = 0.0;
    bool ok = true;
    unsigned c = code;
    for (unsigned i = 0; i < ncand; ++i, c /= nopt) {
      const int l = cand[i];
      const unsigned o = c % nopt;
      if (o == 1) {
        // level 1 (8 nodes of N/8 points) streams through long partial-sum
        // chains and few work items: measured slower than its model, keep it
        // regenerated unless its ranks exceed the solve kernel's capacity
        if (l == 1 && maxr[l] <= kMaxProxyRank) ok = false;
        sbytes += 8.0 * units[l];
        wbytes += 8.0 * (to_half(l) ? ux[l] : units[l]);
      } else if (o == 2) {
        if (l == 1) ok = false;
        sbytes += 8.0 * ux[l];
        wbytes += 8.0 * ux[l];
        evals += units[l] - ux[l];
      } else {
        if (maxr[l] > kMaxProxyRank) ok = false;
        evals += units[l];
        lub += 2.0 * 8.0 * lu[l];  // both orientations read the pair's inverses once
      }
    }
    if (!ok || wbytes > budget) continue;
    const double H = 2.0 * sbytes / kStreamBW;
    const double D = 2.0 * evals / Rp + fixed / Rn + lub / kStreamBW;
    // the factor stream slows both lanes beyond the overlap loss (it pulls
    // the board to its power limit): a term growing with its square,
    // calibrated on C3 (stream vs half level 4, profiles/r02_summary.md)
    const double T = std::max(H, D) + kOverlapLoss * std::min(H, D) + kStreamPower * H * H;
    if (dbg) {
      std::fprintf(stderr, "model");
      unsigned cc = code;
      for (unsigned i = 0; i < ncand; ++i, cc /= nopt) std::fprintf(stderr, " L%d=%u", cand[i], cc % nopt);
      std::fprintf(stderr, "  H %.3f ms D %.3f ms T %.3f ms sbytes %.4g evals %.4g fixed %.4g lub %.4g\n",
                   H * 1e3, D * 1e3, T * 1e3, sbytes, evals, fixed, lub);
    }
    if (T < best) {
      best = T;
      best_code = code;
    }
  }
  if (best == 1e300)
    throw std::runtime_error("initialize: no stream/proxy split fits in device memory");
  unsigned c = best_code;
  for (unsigned i = 0; i < ncand; ++i, c /= nopt) {
    const unsigned o = c % nopt;
    int m = o == 1 ? kModeStream : o == 2 ? kModeHalf : kModeProxy;
    // A large factor stream pulls the board to its power limit and slows both
    // lanes beyond the bandwidth model (C3: 75 GB per matvec, SM clock 1700
    // vs 1965 MHz): stream levels of >= 8 GB per phase go half explicit /
    // half regenerated instead (U' streamed, the other side regenerated, no
    // solves). Measured (profiles/r02_summary.md): C3 level 4 18.3 -> 17.6
    // ms, C4 levels 2 + 4 8.65 -> 8.25 ms, C5 levels 2 + 5 81.5 -> 66.3 ms;
    // C2's 2.3 GB level 3 stays streamed (1.04 vs 1.14 ms half).
    if (m == kModeStream && to_half(cand[i])) m = kModeHalf;
    plan_->set_mode(cand[i], m);
  }
}

// ---------------------------------------------------------------- device plan
void Engine::upload_plan() {
  const Planner& P = *plan_;
  const PlanSizes& Z = P.sizes;
  woff_.upload(P.woff, stream_);
  soff_.upload(P.soff, stream_);
  rowbeg_.upload(P.rowbeg, stream_);
  rpad_.upload(P.rpad, stream_);
  rows_.upload(P.rows, stream_);
  W_.alloc(std::max<std::int64_t>(Z.w_doubles, 2));
  H3D_CUDA_CHECK(cudaMemsetAsync(W_.get(), 0, W_.size() * 8, stream_));
  // + padding: the phase-2 stream consumers prefetch one stage of S ahead
  S_.alloc(std::max<std::int64_t>(Z.s_doubles, 2) + 4 * kTileCols);
  H3D_CUDA_CHECK(cudaMemsetAsync(S_.get(), 0, S_.size() * 8, stream_));
  spos_.upload(P.spos, stream_);
  P_.alloc(std::max<std::int64_t>(Z.p_doubles, 1));
  piv_.alloc(std::max<std::int64_t>(Z.piv_total, 1));
  lu_total_ = Z.lu_total;
  lu_.alloc(std::max<std::int64_t>(2 * Z.lu_total, 1));  // row-major + column-major inverses
  // proxy records share S's index space; padding slots sit far away with
  // weight 0 (see matvec.cu)
  q4_.alloc(4 * std::max<std::int64_t>(Z.s_doubles, 2));
  launch_fill_far(q4_.get(), std::max<std::int64_t>(Z.s_doubles, 2), false, stream_);
  q4c_.alloc(4 * std::max<std::int64_t>(Z.s_doubles, 2));
  launch_fill_far(q4c_.get(), std::max<std::int64_t>(Z.s_doubles, 2), true, stream_);
  center_.upload(P.center, stream_);
  vcols_.upload(P.vcols, stream_);
  std::vector<ProxySeg> solve, solve2;
  for (const auto& s : P.proxy_segs)
    if (s.solve == 2) solve2.push_back(s);
    else if (s.solve) solve.push_back(s);
  std::stable_sort(solve2.begin(), solve2.end(), [](const ProxySeg& a, const ProxySeg& b) { return a.r > b.r; });
  n_segs_solve2_ = static_cast<std::int64_t>(solve2.size());
  segs_solve2_.upload(solve2.empty() ? std::vector<ProxySeg>{ProxySeg{}} : solve2, stream_);
  // largest blocks first: the solve kernel hands segments round-robin to its
  // warps, so the long ones start early and the short ones fill in
  std::stable_sort(solve.begin(), solve.end(), [](const ProxySeg& a, const ProxySeg& b) { return a.r > b.r; });
  n_segs_all_ = static_cast<std::int64_t>(P.proxy_segs.size());
  n_segs_solve_ = static_cast<std::int64_t>(solve.size());
  segs_all_.upload(P.proxy_segs, stream_);
  segs_solve_.upload(solve, stream_);
  // phase-1 items split by resource: HBM-bound stream items and FP64-bound
  // proxy items run as two concurrent persistent kernels
  std::vector<P1Item> si, pi;
  for (const auto& it : P.items) (it.kind == kModeStream ? si : pi).push_back(it);
  p1_stream_items_.upload(si, stream_);
  {
    std::vector<StreamDesc> d(si.size());
    for (std::size_t i = 0; i < si.size(); ++i) {
      const P1Item& it = si[i];
      const int nct = P.rpad[it.node] / kTileCols;
      d[i].wbase = P.woff[it.node] +
                   (static_cast<std::int64_t>(it.row0 / kTileRows) * nct + it.col0 / kTileCols) * kTileDoubles;
      d[i].aux = P.rowbeg[it.node] + it.row0;
      d[i].sbase = 0;
      d[i].nrt = (it.nrows + kTileRows - 1) / kTileRows;
      d[i].ncti = (it.ncols + kTileCols - 1) / kTileCols;
      d[i].nct = nct;
      d[i].nrows = it.nrows;
      d[i].ncols = it.ncols;
      d[i].pad = 0;
    }
    p1s_desc_.upload(d, stream_);
  }
  p1_proxy_items_.upload(pi, stream_);
  n_p1s_ = static_cast<std::int64_t>(si.size());
  n_p1p_ = static_cast<std::int64_t>(pi.size());
  {
    std::vector<P1Reduce> rs, rp, rh;
    for (const auto& r : P.reds) (r.kind == kModeStream ? rs : r.kind == kModeHalf ? rh : rp).push_back(r);
    p1_red_s_.upload(rs, stream_);
    p1_red_p_.upload(rp, stream_);
    p1_red_h_.upload(rh, stream_);
    n_red_s_ = static_cast<std::int64_t>(rs.size());
    n_red_p_ = static_cast<std::int64_t>(rp.size());
    n_red_h_ = static_cast<std::int64_t>(rh.size());
  }
  for (std::size_t x = 0; x + 1 < P.near_off.size(); ++x)
    if (P.near_off[x + 1] - P.near_off[x] > kMaxNearRanges)
      throw std::logic_error("planner: leaf near list longer than the near kernel's range table");
  near_off_.upload(P.near_off, stream_);
  near_ids_.upload(P.near_ids.empty() ? std::vector<std::int32_t>{0} : P.near_ids, stream_);
  near_dense_.upload(P.near_dense, stream_);
  // the cached near field runs the same symmetric pass as the matrix-free
  // one, with the stored values (bitwise-equal results, test_hmatrix.cpp:138-152)
  sym_near_ = true;
  if (sym_near_) {
    for (std::size_t x = 0; x + 1 < P.sym_off.size(); ++x)
      if (P.sym_off[x + 1] - P.sym_off[x] > kMaxNearRanges)
        throw std::logic_error("planner: leaf near list longer than the near kernel's range table");
    sym_off_.upload(P.sym_off, stream_);
    sym_ids_.upload(P.sym_ids.empty() ? std::vector<std::int32_t>{0} : P.sym_ids, stream_);
    sym_cnt_.upload(P.sym_cnt.empty() ? std::vector<std::int32_t>{0} : P.sym_cnt, stream_);
    out_off_.upload(P.out_off, stream_);
    in_off_.upload(P.in_off, stream_);
    in_pos_.upload(P.in_pos.empty() ? std::vector<std::int64_t>{0} : P.in_pos, stream_);
    pairbuf_.alloc(std::max<std::int64_t>(P.out_off.back(), 1));
  }
  has_stream_levels_ = false;
  for (int l = 1; l <= L_; ++l)
    if (P.mode(l) == kModeStream && !P.pairs(l).X.empty()) has_stream_levels_ = true;
  p2_items_.upload(P.p2_items, stream_);
  h2_items_.upload(P.h2_items.empty() ? std::vector<H2Item>{H2Item{}} : P.h2_items, stream_);
  n_h2_ = static_cast<std::int64_t>(P.h2_items.size());
  n_p2_ = static_cast<std::int64_t>(P.p2_items.size());
  p2s_items_.upload(P.p2s_items, stream_);
  {
    std::vector<StreamDesc> d(P.p2s_items.size());
    for (std::size_t i = 0; i < d.size(); ++i) {
      const P2Item& it = P.p2s_items[i];
      const int nct = P.rpad[it.node] / kTileCols;
      d[i].wbase = P.woff[it.node] + static_cast<std::int64_t>(it.row0 / kTileRows) * nct * kTileDoubles;
      d[i].aux = static_cast<std::int64_t>(it.slot) * n_ + P.rowbeg[it.node] + it.row0;
      d[i].sbase = P.soff[it.node];
      d[i].nrt = 1;
      d[i].ncti = nct;
      d[i].nct = nct;
      d[i].nrows = it.nrows;
      d[i].ncols = 0;
      d[i].pad = 0;
    }
    p2s_desc_.upload(d, stream_);
  }
  n_p2s_ = static_cast<std::int64_t>(P.p2s_items.size());
  n_lvl_ = P.n_proxy_levels;
  if (n_lvl_ > 0 || sym_near_) {
    cpart_.alloc(n_);
    // rows of nodes without partners at a level are never written
    lvl_part_.alloc(static_cast<std::size_t>(n_lvl_) * n_);
    H3D_CUDA_CHECK(cudaMemsetAsync(lvl_part_.get(), 0, sizeof(double) * n_lvl_ * n_, stream_));
  }
  // pair levels: descriptors, output runs, gather items, one counter per level
  pair_descs_.upload(P.pair_descs.empty() ? std::vector<PairDesc>{PairDesc{}} : P.pair_descs, stream_);
  pd_level_ = P.pd_level;
  fused_descs_.upload(P.fused_descs.empty() ? std::vector<FusedDesc>{FusedDesc{}} : P.fused_descs, stream_);
  fd_level_ = P.fd_level;
  pg_level_ = P.pg_level;
  // gather items per lane: pair levels on the HBM lane, fused levels on the
  // FP64 lane (each range contiguous: levels of one kind are gathered together
  // only when they are adjacent; otherwise per level, see enqueue)
  pc_off_.upload(P.pc_off, stream_);
  pc_pos_.upload(P.pc_pos.empty() ? std::vector<std::int64_t>{0} : P.pc_pos, stream_);
  pg_items_.upload(P.pg_items.empty() ? std::vector<P2Item>{P2Item{}} : P.pg_items, stream_);
  n_pg_ = static_cast<std::int64_t>(P.pg_items.size());
  pair_out_.alloc(std::max<std::int64_t>(P.pair_out_total, 1));
  counters_.alloc(kCounters);
  sync_flag_.alloc(1);
  H3D_CUDA_CHECK(cudaMemsetAsync(sync_flag_.get(), 0, sizeof(unsigned), stream_));
  if (P.near_storage() != 0) {
    nf_off_.upload(P.nf_off, stream_);
    nf_cols_.upload(P.nf_cols, stream_);
    NF_.alloc(std::max<std::int64_t>(P.nf_total, 1));
  }
  x_.alloc(n_);
  xp_.alloc(n_ + 2);  // + pad: the pair pass bulk-copies x runs rounded to 16 B
  b_.alloc(n_);
  H3D_CUDA_CHECK(cudaStreamSynchronize(stream_));
}

Phase2Args Engine::phase2_args(double* bout) const {
  const Planner& P = *plan_;
  Phase2Args a;
  a.depth = L_;
  a.leaf0 = P.leaf0;
  a.nleaves = P.leaf1 - P.leaf0;
  a.leaf_off = leaf_off_.get();
  a.nt = NodeTable{rowbeg_.get(), rows_.get(), woff_.get(), rpad_.get(), soff_.get()};
  a.W = W_.get();
  a.S = S_.get();
  a.xp = xp_.get();
  a.px = px_.get();
  a.py = py_.get();
  a.pz = pz_.get();
  a.p4 = p4_.get();
  a.q4 = q4_.get();
  a.q4c = q4c_.get();
  a.cen = center_.get();
  a.vcols = vcols_.get();
  a.perm = perm_.get();
  a.near_off = near_off_.get();
  a.near_ids = near_ids_.get();
  a.near_dense = near_dense_.get();
  if (P.near_storage() != 0) {
    a.nf_off = nf_off_.get();
    a.nf_cols = nf_cols_.get();
    a.NF = NF_.get();
    a.nf_mask = P.near_storage();
  }
  a.kernel = opt_.kernel_id;
  a.diag = opt_.diagonal;
  a.b = bout;
  if (n_lvl_ > 0 || sym_near_) {
    a.cpart_out = cpart_.get();
    a.lvl_part = lvl_part_.get();
  }
  if (sym_near_) {
    a.sym_off = sym_off_.get();
    a.sym_ids = sym_ids_.get();
    a.sym_cnt = sym_cnt_.get();
    a.out_off = out_off_.get();
    a.pairbuf = pairbuf_.get();
  }
  if (n_p2s_ > 0) {
    a.p2s_items = p2s_items_.get();
    a.p2s_descs = p2s_desc_.get();
    a.n_p2s_items = n_p2s_;
  }
  if (n_p2_ > 0) {
    a.p2_items = p2_items_.get();
    a.n_p2_items = n_p2_;
    a.lvl_part = lvl_part_.get();
  }
  if (n_h2_ > 0) {
    a.h2_items = h2_items_.get();
    a.n_h2_items = n_h2_;
    a.lvl_part = lvl_part_.get();
    a.spos = spos_.get();
    a.Sw = S_.get();
    a.P = P_.get();
  }
  a.n_total = n_;
  for (int l = 0; l <= L_ && l < 24; ++l) {
    a.lbase[l] = P.node_base()[l];
    a.mode[l] = P.mode(l);
  }
  return a;
}

void Engine::near_scan() {
  const Planner& P = *plan_;
  if (P.leaf1 <= P.leaf0) return;
  Phase2Args a = phase2_args(nullptr);
  if (P.near_storage() == 0) a.nf_off = nullptr;
  H3D_CUDA_CHECK(cudaMemsetAsync(flags_.get(), 0, 4, stream_));
  launch_near_scan(a, P.near_storage() != 0 ? NF_.get() : nullptr, flags_.get(), stream_);
  check_flags("near field");
}

// ---------------------------------------------------------------- matvec
// Enqueue one matvec on stream s: x (original order, device) -> b (original
// order, device). ev (optional, 4 events) brackets gather/exchange, phase 1
// (+ reduce + proxy solves), phase 2. Returns the number of kernels launched.
std::int64_t Engine::enqueue(const double* xin, double* bout, cudaStream_t s, cudaEvent_t* ev,
                            std::uint32_t* kmask) {
  const Planner& P = *plan_;
  std::int64_t launches = 0;
  // profiled calls: a (begin, end) event pair around each kernel on its lane
  auto kb = [&](int k, cudaStream_t st) {
    if (kmask) cudaEventRecord(ev[4 + 2 * k], st);
  };
  auto run = [&](int k) { return !(tune_.skip & (1 << k)); };
  auto ke = [&](int k, cudaStream_t st) {
    if (kmask) {
      cudaEventRecord(ev[5 + 2 * k], st);
      *kmask |= 1u << k;
    }
  };
  if (ev) cudaEventRecord(ev[0], s);
  if (nccl_comm_ == nullptr) {
    // no communicator (one GPU, or a shard built on replicated x): gather
    // all of x locally. With one attached (any world size, including 1 for
    // tests/test_gpu_sharded.py) the exchange below runs.
    kb(H3D_K_GATHER, s);
    launch_gather(xin, perm_.get(), n_, xp_.get(), p4_.get(), s);
    ke(H3D_K_GATHER, s);
    ++launches;
  } else {
    // own slice of x in Morton order, then the all-gather of x over NVLink
    if (P.row1 > P.row0) {
      launch_gather(xin, perm_.get() + P.row0, P.row1 - P.row0, xp_.get() + P.row0,
                    p4_.get() + 4 * P.row0, s);
      ++launches;
    }
    auto comm = static_cast<ncclComm_t>(nccl_comm_);
    NCCL_CHECK(nccl().GroupStart());
    for (int r = 0; r < world_; ++r) {
      const std::int64_t c = P.rank_row1[r] - P.rank_row0[r];
      if (c > 0)
        NCCL_CHECK(nccl().Broadcast(xp_.get() + P.rank_row0[r], xp_.get() + P.rank_row0[r],
                                 static_cast<std::size_t>(c), ncclDouble, r, comm, s));
    }
    NCCL_CHECK(nccl().GroupEnd());
    launch_pack_w(xp_.get(), n_, p4_.get(), s);
    ++launches;
  }
  if (ev) cudaEventRecord(ev[1], s);
  // ---- phase 1: v = K(P, Z) x (proxy levels) / V^T x (stream levels)
  NodeTable nt{rowbeg_.get(), rows_.get(), woff_.get(), rpad_.get(), soff_.get()};
  P1Args a1;
  a1.nt = nt;
  a1.W = W_.get();
  a1.xp = xp_.get();
  a1.spos = spos_.get();
  a1.S = S_.get();
  a1.P = P_.get();
  a1.px = px_.get();
  a1.py = py_.get();
  a1.pz = pz_.get();
  a1.p4 = p4_.get();
  a1.q4 = q4_.get();
  a1.q4c = q4c_.get();
  a1.cen = center_.get();
  a1.vcols = vcols_.get();
  // Two lanes forked from s, joined back for the combine:
  //   stream2_ (HBM): p1_stream -> stream reductions -> [solves done] -> p2_stream
  //   stream4_ (FP64): p1_proxy -> proxy reductions -> solves -> p2_proxy ->
  //            near field + direct leaf blocks
  // Persistent CTAs with per-SM budgets: one 5-warp bulk-copy CTA per SM holds
  // HBM near peak, the FP64 kernels fill the remaining registers.
  const bool has_p2 = P.leaf1 > P.leaf0;
  const bool parts = n_lvl_ > 0 || sym_near_;  // near pass writes partials, combine sums them
  // (with a 1-rank communicator the gather runs too: the path is exercised on one GPU)
  const bool gather_b = (opt_.gather_b != 0 || force_gather_) && nccl_comm_ != nullptr;
  if (opt_.gather_b != 0 && nccl_comm_ == nullptr && world_ > 1)
    throw InvalidArgument("matvec: gather_b needs a communicator (attach_nccl) on a sharded handle");
  const bool pair_lv = pd_level_.size() > 1 && pd_level_.back() > 0;
  const bool hbm = n_p1s_ > 0 || n_p2s_ > 0 || pair_lv;
  const bool fused_lv = fd_level_.size() > 1 && fd_level_.back() > 0;
  const bool fp = n_p1p_ > 0 || n_segs_solve_ > 0 || n_p2_ > 0 || fused_lv || n_h2_ > 0;
  // per-level gather of pair-major outputs into the level partials
  auto gather_levels = [&](int mode, cudaStream_t st) {
    for (int l = 1; l <= L_; ++l) {
      if (P.mode(l) != mode) continue;
      const std::int64_t g0 = pg_level_[l], g1 = pg_level_[l + 1];
      if (g1 <= g0) continue;
      launch_pair_gather(pg_items_.get() + g0, g1 - g0, rowbeg_.get(), pc_off_.get(), pc_pos_.get(),
                         pair_out_.get(), lvl_part_.get(), n_, st);
      ++launches;
    }
  };
  H3D_CUDA_CHECK(cudaMemsetAsync(counters_.get(), 0, kCounters * sizeof(unsigned), s));
  H3D_CUDA_CHECK(cudaMemsetAsync(sync_flag_.get(), 0, sizeof(unsigned), s));
  Phase2Args a2 = phase2_args(bout);
  a2.counter = counters_.get() + 2;
  a2.counter2 = counters_.get() + 3;
  a2.counter3 = counters_.get() + 4;
  H3D_CUDA_CHECK(cudaEventRecord(fork_[0], s));
  // HBM lane: pair levels (one fused read per pair, x only), phase 1
  if (hbm) {
    H3D_CUDA_CHECK(cudaStreamWaitEvent(stream2_, fork_[0], 0));
    if (pair_lv && has_p2) {
      kb(H3D_K_PAIR, stream2_);
      for (int l = 1; l <= L_; ++l) {
        const std::int64_t n = pd_level_[l + 1] - pd_level_[l];
        if (n == 0) continue;
        PairArgs pa;
        pa.descs = pair_descs_.get() + pd_level_[l];
        pa.n = n;
        pa.W = W_.get();
        pa.xp = xp_.get();
        pa.out = pair_out_.get();
        launch_pair(pa, sms_, tune_.pps > 0 ? tune_.pps : 2, stream2_);
        ++launches;
      }
      gather_levels(kModePair, stream2_);
      ke(H3D_K_PAIR, stream2_);
    }
    if (n_p1s_ > 0) {
      a1.items = p1_stream_items_.get();
      a1.descs = p1s_desc_.get();
      a1.nitems = n_p1s_;
      a1.counter = counters_.get();
      kb(H3D_K_P1_STREAM, stream2_);
      if (run(H3D_K_P1_STREAM)) launch_p1_stream(a1, sms_, fp ? tune_.p1s : 2, stream2_);
      ke(H3D_K_P1_STREAM, stream2_);
      ++launches;
    }
    if (n_red_s_ > 0) {
      kb(H3D_K_RED_STREAM, stream2_);
      launch_phase1_reduce(p1_red_s_.get(), n_red_s_, nt, spos_.get(), P_.get(), S_.get(), stream2_);
      ke(H3D_K_RED_STREAM, stream2_);
      ++launches;
    }
    // phase 1 of the HBM lane done: p2_stream is next on this lane
    H3D_CUDA_CHECK(cudaEventRecord(fork_[1], stream2_));
  }
  // FP64 lane: phase 1 proxy levels -> reductions -> solves
  H3D_CUDA_CHECK(cudaStreamWaitEvent(stream4_, fork_[0], 0));
  if (n_p1p_ > 0) {
    a1.items = p1_proxy_items_.get();
    a1.nitems = n_p1p_;
    a1.counter = counters_.get() + 1;
    kb(H3D_K_P1_PROXY, stream4_);
    if (run(H3D_K_P1_PROXY)) launch_p1_proxy(a1, opt_.kernel_id, sms_, hbm ? tune_.p1p : 8, stream4_);
    ke(H3D_K_P1_PROXY, stream4_);
    ++launches;
  }
  // the near field + direct leaf blocks (x only) fork off here, beside the
  // latency-bound solves (H3D_TUNE nf=0: after p2_proxy on the FP64 lane).
  // Measured with the batched-load solve: C2 / C3 / C4 3.5-5.5 % faster
  // (before it the solves lost more than the near field gained)
  // the near field (x only) forks beside the latency-bound solves
  const int nf_mode = tune_.nf >= 0 ? tune_.nf : (n_h2_ > 0 ? 2 : 1);
  const bool near_fork = has_p2 && nf_mode != 0;
  auto fork_near = [&] {
    H3D_CUDA_CHECK(cudaEventRecord(fork_[2], stream4_));
    H3D_CUDA_CHECK(cudaStreamWaitEvent(stream3_, fork_[2], 0));
    kb(H3D_K_NEAR, stream3_);
    if (run(H3D_K_NEAR)) launch_p2_near(a2, sms_, tune_.nfc, stream3_);
    ke(H3D_K_NEAR, stream3_);
    ++launches;
    H3D_CUDA_CHECK(cudaEventRecord(join_[2], stream3_));
  };
  // nf 1: right after p1_proxy; nf 2 (default with a two-use pass): after
  // that pass, so the near field overlaps the solves and p2_proxy as before
  if (near_fork && nf_mode == 1) fork_near();
  if (n_red_p_ > 0) {
    kb(H3D_K_RED_PROXY, stream4_);
    launch_phase1_reduce(p1_red_p_.get(), n_red_p_, nt, spos_.get(), P_.get(), S_.get(), stream4_);
    ke(H3D_K_RED_PROXY, stream4_);
    ++launches;
  }
  // half levels, the regenerated side: both uses per entry in one pass, once
  // the partners' streamed phase 1 (its t) is in S; p2_stream waits for its v
  const bool h2 = n_h2_ > 0 && has_p2;
  if (h2 && n_segs_solve2_ > 0) {
    // split levels: the Y-role columns' weights are solved before the pass
    kb(H3D_K_SOLVE, stream4_);
    launch_proxy_solve(segs_solve2_.get(), n_segs_solve2_, lu_.get(), lu_total_, S_.get(), sms_, tune_.sol,
                       counters_.get() + 7, stream4_);
    ke(H3D_K_SOLVE, stream4_);
    ++launches;
  }
  if (h2) {
    if (hbm && tune_.h2w) H3D_CUDA_CHECK(cudaStreamWaitEvent(stream4_, fork_[1], 0));
    kb(H3D_K_HALF, stream4_);
    a2.counter_h2 = counters_.get() + 6;
    launch_half2(a2, sms_, hbm ? tune_.p2p : 8, stream4_);
    if (n_red_h_ > 0)
      launch_phase1_reduce(p1_red_h_.get(), n_red_h_, nt, spos_.get(), P_.get(), S_.get(), stream4_);
    ke(H3D_K_HALF, stream4_);
    launches += 1 + (n_red_h_ > 0 ? 1 : 0);
    H3D_CUDA_CHECK(cudaEventRecord(h2_done_, stream4_));
  }
  if (near_fork && nf_mode == 2) fork_near();
  if (n_segs_solve_ > 0) {
    kb(H3D_K_SOLVE, stream4_);
    launch_proxy_solve(segs_solve_.get(), n_segs_solve_, lu_.get(), lu_total_, S_.get(), sms_, tune_.sol,
                       counters_.get() + 5, stream4_);
    ke(H3D_K_SOLVE, stream4_);
    ++launches;
  }
  if (ev) cudaEventRecord(ev[2], stream4_);
  // HBM lane, phase 2: launched right behind phase 1 so its CTAs take the
  // SM slots p1_stream leaves (a persistent FP64 kernel launched first would
  // crowd them out for its whole run), but its producer holds the first copy
  // until the FP64 lane flags the solves done: the latency-bound solve
  // blocks lose most of their bandwidth beside a saturating bulk stream
  // (0.5 ms alone vs 6-10 ms beside it), and they gate the FP64 lane.
  if (hbm) {
    if (n_segs_solve_ > 0 && has_p2 && n_p2s_ > 0 && tune_.fw) {
      launch_set_flag(sync_flag_.get(), 1u, stream4_);
      ++launches;
      a2.wait_flag = sync_flag_.get();
      a2.wait_value = 1u;
    }
    if (h2) H3D_CUDA_CHECK(cudaStreamWaitEvent(stream2_, h2_done_, 0));
    if (has_p2 && n_p2s_ > 0) {
      kb(H3D_K_P2_STREAM, stream2_);
      if (run(H3D_K_P2_STREAM)) launch_p2_stream(a2, sms_, fp ? tune_.p2s : 2, stream2_);
      ke(H3D_K_P2_STREAM, stream2_);
      ++launches;
    }
    H3D_CUDA_CHECK(cudaEventRecord(join_[0], stream2_));
  }
  // FP64 lane, phase 2: proxy levels, then the near field + direct leaf
  // blocks (one persistent FP64 kernel resident at a time next to the HBM
  // lane's bulk-copy CTA)
  if (has_p2) {
    // the FP64 lane's persistent phase-2 kernels start only once the HBM
    // lane's phase 1 is done, so p2_stream (launched first) takes its SM slots
    // before them: when the solves finish early, a p2_proxy launched ahead of
    // p2_stream holds the SMs for its whole run and the stream loses
    // bandwidth (measured: C3 p2_stream 10.3 -> 12.3 ms)
    if (hbm && tune_.p2o) H3D_CUDA_CHECK(cudaStreamWaitEvent(stream4_, fork_[1], 0));
    if (fused_lv) {
      kb(H3D_K_FUSED, stream4_);
      FusedArgs fa;
      fa.descs = fused_descs_.get();
      fa.n = fd_level_.back();
      fa.p4 = p4_.get();
      fa.piv = piv_.get();
      fa.lu = lu_.get();
      fa.lu_total = lu_total_;
      fa.out = pair_out_.get();
      if (run(H3D_K_FUSED)) launch_fused(fa, opt_.kernel_id, sms_, stream4_);
      ++launches;
      gather_levels(kModeFused, stream4_);
      ke(H3D_K_FUSED, stream4_);
    }
    if (n_p2_ > 0) {
      kb(H3D_K_P2_PROXY, stream4_);
      if (run(H3D_K_P2_PROXY)) launch_p2_proxy(a2, sms_, hbm ? tune_.p2p : 8, stream4_);
      ke(H3D_K_P2_PROXY, stream4_);
      ++launches;
    }
    if (!near_fork) {
      kb(H3D_K_NEAR, stream4_);
      if (run(H3D_K_NEAR)) launch_p2_near(a2, sms_, hbm ? tune_.p2c : 4, stream4_);
      ke(H3D_K_NEAR, stream4_);
      ++launches;
    }
  }
  H3D_CUDA_CHECK(cudaEventRecord(join_[1], stream4_));
  H3D_CUDA_CHECK(cudaStreamWaitEvent(s, join_[1], 0));
  if (near_fork) H3D_CUDA_CHECK(cudaStreamWaitEvent(s, join_[2], 0));
  if (hbm) H3D_CUDA_CHECK(cudaStreamWaitEvent(s, join_[0], 0));
  if (has_p2 && parts) {
    kb(H3D_K_COMBINE, s);
    launch_combine(cpart_.get(), lvl_part_.get(), n_lvl_, n_, leaf_off_.get(), P.leaf0, P.leaf1 - P.leaf0,
                   sym_near_ ? in_off_.get() : nullptr, sym_near_ ? in_pos_.get() : nullptr,
                   sym_near_ ? pairbuf_.get() : nullptr, perm_.get(), bout,
                   gather_b ? bm_.get() : nullptr, s);
    ke(H3D_K_COMBINE, s);
    ++launches;
  }
  if (gather_b) {
    // the full b on every rank (parallel.cpp:284-290): each rank's owned
    // Morton slice to all, then the other ranks' rows to the original order
    auto comm = static_cast<ncclComm_t>(nccl_comm_);
    NCCL_CHECK(nccl().GroupStart());
    for (int r = 0; r < world_; ++r) {
      const std::int64_t c = P.rank_row1[r] - P.rank_row0[r];
      if (c > 0)
        NCCL_CHECK(nccl().Broadcast(bm_.get() + P.rank_row0[r], bm_.get() + P.rank_row0[r],
                                 static_cast<std::size_t>(c), ncclDouble, r, comm, s));
    }
    NCCL_CHECK(nccl().GroupEnd());
    launch_unpermute_rest(bm_.get(), perm_.get(), n_, P.row0, P.row1, bout, s);
    ++launches;
  }
  if (nccl_comm_ != nullptr) ++comm_matvecs_;
  if (ev) cudaEventRecord(ev[3], s);
  return launches;
}

void Engine::begin_call(cudaStream_t s) {
  if (done_valid_ && s != last_stream_) H3D_CUDA_CHECK(cudaStreamWaitEvent(s, done_ev_, 0));
}

void Engine::end_call(cudaStream_t s) {
  H3D_CUDA_CHECK(cudaEventRecord(done_ev_, s));
  done_valid_ = true;
  last_stream_ = s;
}

void Engine::matvec(const double* x, double* b, bool host, h3d_timing* t) {
  H3D_CUDA_CHECK(cudaSetDevice(opt_.device));
  begin_call(stream_);
  cudaEventRecord(ev_[0], stream_);
  const double* xin = x;
  if (host) {
    H3D_CUDA_CHECK(cudaMemcpyAsync(x_.get(), x, n_ * 8, cudaMemcpyHostToDevice, stream_));
    xin = x_.get();
  }
  double* bout = host ? b_.get() : b;
  // through the graph cache (events around it: copies and device time), or
  // eagerly with per-phase events when graphs are off (H3D_TUNE graphs=0)
  // or a communicator is attached
  const bool graphed = tune_.graphs && nccl_comm_ == nullptr;
  std::int64_t launches = 0;
  if (graphed) {
    cudaEventRecord(ev_[1], stream_);
    launches = run_graph(xin, bout, stream_);
    cudaEventRecord(ev_[4], stream_);
  } else {
    launches = enqueue(xin, bout, stream_, ev_ + 1, nullptr);
  }
  if (host) H3D_CUDA_CHECK(cudaMemcpyAsync(b, b_.get(), n_ * 8, cudaMemcpyDeviceToHost, stream_));
  cudaEventRecord(ev_[5], stream_);
  end_call(stream_);
  H3D_CUDA_CHECK(cudaStreamSynchronize(stream_));
  if (t) {
    float v = 0;
    auto el = [&](int a, int bb) {
      cudaEventElapsedTime(&v, ev_[a], ev_[bb]);
      return static_cast<double>(v);
    };
    std::memset(t, 0, sizeof(*t));
    t->total_ms = el(0, 5);
    t->h2d_ms = el(0, 1);
    t->d2h_ms = el(4, 5);
    if (graphed) {
      t->device_ms = el(1, 4);  // one graph: no per-phase split
    } else {
      if (world_ == 1) t->gather_ms = el(1, 2);
      else t->exchange_ms = el(1, 2);
      t->phase1_ms = el(2, 3);
      t->phase2_ms = el(3, 4);
      t->device_ms = el(1, 4);
    }
    t->launches = launches;
  }
}

// Replay of the captured matvec for (x, b): the first call runs eagerly (it
// also sets the kernels' one-time attributes), the second captures the whole
// two-lane enqueue on the engine's stream (fork / join through events become
// graph edges) and every later call is one cudaGraphLaunch on the caller's
// stream. Not used with a communicator attached, with profiling on, or with
// H3D_TUNE graphs=0.
std::int64_t Engine::run_graph(const double* x, double* b, cudaStream_t s) {
  if (!tune_.graphs || nccl_comm_ != nullptr) return enqueue(x, b, s, nullptr, nullptr);
  GraphEntry* e = nullptr;
  for (auto& g : graphs_)
    if (g.x == x && g.b == b) e = &g;
  if (e == nullptr) {
    if (graphs_.size() >= 8) {
      if (graphs_.front().exec) cudaGraphExecDestroy(graphs_.front().exec);
      graphs_.erase(graphs_.begin());
    }
    graphs_.push_back(GraphEntry{x, b, nullptr, 0, 0});
    e = &graphs_.back();
  }
  if (e->exec == nullptr) {
    if (e->seen++ == 0) return enqueue(x, b, s, nullptr, nullptr);
    H3D_CUDA_CHECK(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeRelaxed));
    std::int64_t launches = 0;
    try {
      launches = enqueue(x, b, stream_, nullptr, nullptr);
    } catch (...) {
      cudaGraph_t g = nullptr;
      cudaStreamEndCapture(stream_, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    cudaGraph_t g = nullptr;
    H3D_CUDA_CHECK(cudaStreamEndCapture(stream_, &g));
    const cudaError_t err = cudaGraphInstantiate(&e->exec, g, 0);
    cudaGraphDestroy(g);
    H3D_CUDA_CHECK(err);
    e->launches = launches;
  }
  H3D_CUDA_CHECK(cudaGraphLaunch(e->exec, s));
  return e->launches;
}

void Engine::matvec_async(const double* x, double* b, cudaStream_t s) {
  H3D_CUDA_CHECK(cudaSetDevice(opt_.device));
  begin_call(s);
  if (!prof_on_) {
    prof_launches_ += run_graph(x, b, s);
    end_call(s);
    return;
  }
  cudaEvent_t* ev = nullptr;
  std::uint32_t* mask = nullptr;
  if (prof_on_) {
    if (prof_used_ >= prof_ev_.size() / kProfEv) throw InvalidArgument("profile ring full; read it first");
    ev = prof_ev_.data() + kProfEv * prof_used_;
    mask = prof_mask_.data() + prof_used_;
    *mask = 0;
    ++prof_used_;
  }
  prof_launches_ += enqueue(x, b, s, ev, mask);
  end_call(s);
}

void Engine::profile(int enable, std::int64_t capacity) {
  H3D_CUDA_CHECK(cudaSetDevice(opt_.device));
  prof_on_ = enable != 0;
  prof_used_ = 0;
  prof_launches_ = 0;
  const std::size_t cap = static_cast<std::size_t>(std::max<std::int64_t>(capacity, 1));
  if (prof_on_ && prof_ev_.size() < kProfEv * cap) {
    for (auto e : prof_ev_) cudaEventDestroy(e);
    prof_ev_.assign(kProfEv * cap, nullptr);
    for (auto& e : prof_ev_) H3D_CUDA_CHECK(cudaEventCreate(&e));
  }
  if (prof_on_ && prof_mask_.size() < cap) prof_mask_.assign(cap, 0u);
}

void Engine::profile_read(h3d_timing* sum, std::int64_t* steps) {
  H3D_CUDA_CHECK(cudaSetDevice(opt_.device));
  std::memset(sum, 0, sizeof(*sum));
  for (int q = 0; q < H3D_K_COUNT; ++q) {
    prof_kms_[q] = 0.0;
    prof_kstart_[q] = 0.0;
    prof_kn_[q] = 0;
  }
  for (std::size_t k = 0; k < prof_used_; ++k) {
    cudaEvent_t* ev = prof_ev_.data() + kProfEv * k;
    H3D_CUDA_CHECK(cudaEventSynchronize(ev[3]));
    for (int q = 0; q < H3D_K_COUNT; ++q) {
      if (!(prof_mask_[k] & (1u << q))) continue;
      float d = 0;
      H3D_CUDA_CHECK(cudaEventSynchronize(ev[5 + 2 * q]));
      cudaEventElapsedTime(&d, ev[4 + 2 * q], ev[5 + 2 * q]);
      prof_kms_[q] += d;
      float o = 0;
      cudaEventElapsedTime(&o, ev[0], ev[4 + 2 * q]);
      prof_kstart_[q] += o;
      ++prof_kn_[q];
    }
    float a = 0, b = 0, c = 0;
    cudaEventElapsedTime(&a, ev[0], ev[1]);
    cudaEventElapsedTime(&b, ev[1], ev[2]);
    cudaEventElapsedTime(&c, ev[2], ev[3]);
    if (world_ == 1) sum->gather_ms += a;
    else sum->exchange_ms += a;
    sum->phase1_ms += b;
    sum->phase2_ms += c;
    sum->total_ms += a + b + c;
    sum->device_ms += a + b + c;
  }
  sum->launches = prof_launches_;
  *steps = static_cast<std::int64_t>(prof_used_);
  prof_used_ = 0;
  prof_launches_ = 0;
}

void Engine::profile_kernels(double* ms_sum, std::int64_t* launches, double* start_sum,
                             int count) const {
  for (int q = 0; q < count && q < H3D_K_COUNT; ++q) {
    ms_sum[q] = prof_kms_[q];
    launches[q] = prof_kn_[q];
    if (start_sum) start_sum[q] = prof_kstart_[q];
  }
}

void Engine::attach_nccl(const void* id128, int rank, int world) {
  if (world != world_ || rank != rank_)
    throw InvalidArgument("attach_nccl: rank/world differ from the engine's shard options");
  H3D_CUDA_CHECK(cudaSetDevice(opt_.device));
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  ncclComm_t comm;
  NCCL_CHECK(nccl().CommInitRank(&comm, world, id, rank));
  nccl_comm_ = comm;
  if (opt_.gather_b != 0) bm_.alloc(static_cast<std::size_t>(n_));
  // captured graphs of an unattached handle must not be replayed (no exchange)
  for (auto& g : graphs_)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  graphs_.clear();
}

void Engine::comm_ledger(h3d_comm_ledger* out) const {
  std::memset(out, 0, sizeof(*out));
  if (nccl_comm_ == nullptr) return;
  const Planner& P = *plan_;
  const std::int64_t owned = P.row1 - P.row0;
  int slices = 0;
  for (int r = 0; r < world_; ++r) slices += P.rank_row1[r] > P.rank_row0[r] ? 1 : 0;
  out->x_gather_doubles = n_ - owned;
  out->b_gather_doubles = opt_.gather_b != 0 ? n_ - owned : 0;
  out->collectives = slices * (opt_.gather_b != 0 ? 2 : 1);
  out->matvecs = comm_matvecs_;
}

void Engine::stats(h3d_stats* s) const {
  const Planner& P = *plan_;
  const PlanSizes& Z = P.sizes;
  std::memset(s, 0, sizeof(*s));
  s->depth = L_;
  s->max_rank = Z.max_rank;
  s->n = n_;
  s->lowrank_blocks = Z.nblocks_ordered;
  s->aca_pairs = Z.npairs;
  s->sum_rank = Z.sum_rank;
  s->factor_doubles = Z.factor_doubles;
  s->factor_bytes_alloc = Z.w_doubles * 8;
  s->tvec_doubles = Z.s_doubles;
  s->near_blocks = Z.near_blocks;
  s->near_entries = Z.near_entries;
  s->near_bytes_stored = P.near_storage() != 0 ? P.nf_total * 8 : 0;
  // reference RepStats convention (hmatrix.cpp:228-251): r^2 per ordered
  // block + dense leaf areas (directly evaluated leaf blocks count as dense)
  s->ref_float_count = Z.ref_float_count + static_cast<std::uint64_t>(Z.near_entries + Z.direct_evals);
  s->ref_int_count = Z.ref_int_count;
  s->compression_ratio = static_cast<double>(s->ref_float_count) /
                         (static_cast<double>(n_) * static_cast<double>(n_));
  s->build_ms_tree = ms_tree_;
  s->build_ms_lists = ms_lists_;
  s->build_ms_aca_rank = ms_aca_rank_;
  s->build_ms_aca_write = ms_aca_write_;
  s->build_ms_total = ms_total_;
  s->build_ms_plan = ms_plan_;
  s->build_ms_post = ms_post_;
  s->build_ms_near = ms_near_;
  s->phase1_items = n_p1s_ + n_p1p_;
  s->owned_row_begin = P.row0;
  s->owned_row_end = P.row1;
  for (int l = 0; l <= L_ && l < 16; ++l) s->level_modes[l] = P.mode(l);
  s->proxy_units = Z.proxy_units;
  s->half_units = Z.half_units;
  s->direct_evals = Z.direct_evals;
  s->lu_doubles = Z.lu_total;
  for (int l = 1; l <= L_ && l < 16; ++l) {
    const auto& pr = P.pairs(l);
    std::int64_t u = 0;
    for (std::size_t p = 0; p < pr.X.size(); ++p)
      u += static_cast<std::int64_t>(pr.rank[p]) * (node_size(l, pr.X[p]) + node_size(l, pr.Y[p]));
    s->level_units[l] = u;
    s->level_aca_ms[l] = level_aca_ms_[l];
  }
}

void Engine::export_tree(std::int32_t* perm, int level, std::int64_t* offsets) const {
  if (perm) std::memcpy(perm, perm_h_.data(), perm_h_.size() * 4);
  if (offsets) {
    if (level < 0 || level > L_) throw InvalidArgument("export_tree: level out of range");
    std::memcpy(offsets, off_[level].data(), off_[level].size() * 8);
  }
}

std::int64_t Engine::export_list(int level, int kind, std::int32_t* offsets,
                                 std::int32_t* ids) const {
  if (level < 0 || level > L_ || kind < 0 || kind >= kListKinds)
    throw InvalidArgument("export_list: level/kind out of range");
  const auto& o = lists_[level].off[kind];
  const auto& v = lists_[level].ids[kind];
  if (offsets) {
    if (level == 0) {
      offsets[0] = offsets[1] = 0;
    } else {
      std::memcpy(offsets, o.data(), o.size() * 4);
    }
  }
  if (ids && !v.empty()) std::memcpy(ids, v.data(), v.size() * 4);
  return static_cast<std::int64_t>(v.size());
}

std::int64_t Engine::export_pairs(int level, std::int32_t* x, std::int32_t* y,
                                  std::int32_t* rank) const {
  if (level < 1 || level > L_) return 0;
  const auto& P = plan_->pairs(level);
  if (x) std::memcpy(x, P.X.data(), P.X.size() * 4);
  if (y) std::memcpy(y, P.Y.data(), P.Y.size() * 4);
  if (rank) std::memcpy(rank, P.rank.data(), P.rank.size() * 4);
  return static_cast<std::int64_t>(P.X.size());
}

}  // namespace h3db

namespace h3db {

// ---------------------------------------------------------------- solver
void Engine::direct_matvec(const double* x, double* b, bool host) {
  H3D_CUDA_CHECK(cudaSetDevice(opt_.device));
  // every point is resident on every shard: the exact product runs whole here
  begin_call(stream_);
  const double* xin = x;
  if (host) {
    H3D_CUDA_CHECK(cudaMemcpyAsync(x_.get(), x, n_ * 8, cudaMemcpyHostToDevice, stream_));
    xin = x_.get();
  }
  double* bout = host ? b_.get() : b;
  launch_gather(xin, perm_.get(), n_, xp_.get(), p4_.get(), stream_);
  launch_direct(p4_.get(), n_, opt_.kernel_id, opt_.diagonal, perm_.get(), bout, stream_);
  if (host) H3D_CUDA_CHECK(cudaMemcpyAsync(b, b_.get(), n_ * 8, cudaMemcpyDeviceToHost, stream_));
  end_call(stream_);
  H3D_CUDA_CHECK(cudaStreamSynchronize(stream_));
}

double Engine::reference_error(const double* x, const double* b, bool host, std::int64_t exact_limit,
                               std::int64_t sample_rows, std::uint64_t seed) {
  H3D_CUDA_CHECK(cudaSetDevice(opt_.device));
  if (exact_limit < 0 || sample_rows < 0) throw InvalidArgument("reference_error: negative row count");
  // rows are permuted (Morton) positions, drawn exactly as hmatrix.cpp:264-271
  std::vector<std::int64_t> rows;
  if (n_ <= exact_limit) {
    rows.resize(static_cast<std::size_t>(n_));
    for (std::int64_t i = 0; i < n_; ++i) rows[static_cast<std::size_t>(i)] = i;
  } else {
    std::mt19937_64 gen(seed);
    rows.resize(static_cast<std::size_t>(sample_rows));
    for (auto& r : rows)
      r = static_cast<std::int64_t>(static_cast<std::size_t>(static_cast<double>(gen() >> 11) * 0x1.0p-53 *
                                                             static_cast<double>(n_)));
  }
  const std::int64_t nr = static_cast<std::int64_t>(rows.size());
  std::vector<double> exact(rows.size()), bh;
  begin_call(stream_);
  const double* xin = x;
  if (host) {
    H3D_CUDA_CHECK(cudaMemcpyAsync(x_.get(), x, n_ * 8, cudaMemcpyHostToDevice, stream_));
    xin = x_.get();
  } else {
    bh.resize(static_cast<std::size_t>(n_));
    H3D_CUDA_CHECK(cudaMemcpyAsync(bh.data(), b, n_ * 8, cudaMemcpyDeviceToHost, stream_));
  }
  launch_gather(xin, perm_.get(), n_, xp_.get(), p4_.get(), stream_);
  DevBuf<std::int64_t> rows_d;
  DevBuf<double> out_d;
  if (nr > 0) {
    rows_d.upload(rows, stream_);
    out_d.alloc(static_cast<std::size_t>(nr));
    H3D_CUDA_CHECK(cudaMemsetAsync(flags_.get(), 0, 4, stream_));
    launch_exact_rows(p4_.get(), n_, opt_.kernel_id, opt_.diagonal, rows_d.get(), nr, out_d.get(), flags_.get(),
                      stream_);
    H3D_CUDA_CHECK(cudaMemcpyAsync(exact.data(), out_d.get(), nr * 8, cudaMemcpyDeviceToHost, stream_));
  }
  end_call(stream_);
  H3D_CUDA_CHECK(cudaStreamSynchronize(stream_));
  if (nr > 0) check_flags("reference_error");
  const double* bb = host ? b : bh.data();
  double err2 = 0.0, ref2 = 0.0;
  for (std::int64_t k = 0; k < nr; ++k) {
    const double e = exact[static_cast<std::size_t>(k)];
    const double a = bb[perm_h_[static_cast<std::size_t>(rows[static_cast<std::size_t>(k)])]];
    err2 += (a - e) * (a - e);
    ref2 += e * e;
  }
  return std::sqrt(err2 / ref2);
}

void Engine::gmres(const double* rhs, double* xout, bool host, double alpha, double beta, double tol,
                   int restart, int max_iter, double* hist, int hist_cap, h3d_gmres_info* info) {
  H3D_CUDA_CHECK(cudaSetDevice(opt_.device));
  if (!(tol > 0)) throw InvalidArgument("gmres: tol must be positive");
  // sharded handles: the Krylov vectors are replicated on every rank and each
  // operator application all-gathers b (force_gather_), so every rank runs
  // the same deterministic iteration on full vectors
  if (world_ != 1 && nccl_comm_ == nullptr)
    throw InvalidArgument("gmres: a sharded handle needs its communicator (attach_nccl)");
  struct GatherScope {
    Engine* e;
    explicit GatherScope(Engine* en) : e(en) {
      if (e->nccl_comm_ != nullptr && e->bm_.size() == 0) e->bm_.alloc(static_cast<std::size_t>(e->n_));
      e->force_gather_ = e->nccl_comm_ != nullptr;
    }
    ~GatherScope() { e->force_gather_ = false; }
  } gather_scope(this);
  const auto t0 = Clock::now();
  const std::int64_t n = n_;
  max_iter = std::max(max_iter, 1);
  restart = restart > 0 ? restart : max_iter;
  const int mcap = std::min(restart, max_iter);
  cudaStream_t s = stream_;
  begin_call(s);
  DevBuf<double> f, x, w, r, basis, scal, scratch;
  f.alloc(n);
  x.alloc(n);
  w.alloc(n);
  r.alloc(n);
  basis.alloc(static_cast<std::size_t>(mcap + 1) * n);
  scal.alloc(mcap + 2);
  scratch.alloc(dot_scratch_doubles());
  H3D_CUDA_CHECK(cudaMemcpyAsync(f.get(), rhs, n * 8, host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, s));
  H3D_CUDA_CHECK(cudaMemsetAsync(x.get(), 0, n * 8, s));
  auto op = [&](const double* v, double* out) {  // out = alpha v + beta A v
    enqueue(v, out, s, nullptr, nullptr);
    if (!(alpha == 0.0 && beta == 1.0)) launch_affine(out, v, n, alpha, beta, s);
  };
  auto norm_host = [&](const double* v) {
    launch_dot(v, v, n, scratch.get(), scal.get(), true, s);
    double h = 0;
    H3D_CUDA_CHECK(cudaMemcpyAsync(&h, scal.get(), 8, cudaMemcpyDeviceToHost, s));
    H3D_CUDA_CHECK(cudaStreamSynchronize(s));
    return h;
  };
  int hlen = 0, total = 0;
  bool converged = false;
  double relres = 1.0;
  const double rhs_norm = norm_host(f.get());
  if (rhs_norm == 0.0) {
    converged = true;
    relres = 0.0;
  }
  std::vector<double> hcol(mcap + 2);
  while (!converged && total < max_iter) {
    // residual of the current iterate (the rhs itself on the first pass)
    if (total == 0) {
      H3D_CUDA_CHECK(cudaMemcpyAsync(r.get(), f.get(), n * 8, cudaMemcpyDeviceToDevice, s));
    } else {
      op(x.get(), w.get());
      launch_sub(r.get(), f.get(), w.get(), n, s);
    }
    const double beta0 = norm_host(r.get());
    if (beta0 / rhs_norm < tol) {
      converged = true;
      relres = beta0 / rhs_norm;
      break;
    }
    const int m = std::min(restart, max_iter - total);
    H3D_CUDA_CHECK(cudaMemsetAsync(basis.get(), 0, n * 8, s));
    launch_axpy(basis.get(), r.get(), n, nullptr, 0.0, 1.0 / beta0, s);
    std::vector<double> H(static_cast<std::size_t>(m + 1) * m, 0.0), cs(m), sn(m), g(m + 1, 0.0);
    auto Hk = [&](int i, int k) -> double& { return H[static_cast<std::size_t>(i) * m + k]; };
    g[0] = beta0;
    int k = 0;
    bool done = false;
    for (; k < m && !done; ++k) {
      double* vk = basis.get() + static_cast<std::int64_t>(k) * n;
      op(vk, w.get());
      for (int i = 0; i <= k; ++i) {  // modified Gram-Schmidt
        const double* vi = basis.get() + static_cast<std::int64_t>(i) * n;
        launch_dot(w.get(), vi, n, scratch.get(), scal.get() + i, false, s);
        launch_axpy(w.get(), vi, n, scal.get() + i, -1.0, 0.0, s);
      }
      launch_dot(w.get(), w.get(), n, scratch.get(), scal.get() + k + 1, true, s);
      H3D_CUDA_CHECK(cudaMemcpyAsync(hcol.data(), scal.get(), (k + 2) * 8, cudaMemcpyDeviceToHost, s));
      H3D_CUDA_CHECK(cudaStreamSynchronize(s));
      const double h_next = hcol[k + 1];
      if (h_next > 0.0 && k + 1 <= mcap)
        launch_scale_div(basis.get() + static_cast<std::int64_t>(k + 1) * n, w.get(), n,
                         scal.get() + k + 1, s);
      for (int i = 0; i <= k; ++i) Hk(i, k) = hcol[i];
      Hk(k + 1, k) = h_next;
      for (int i = 0; i < k; ++i) {  // previous rotations
        const double t = cs[i] * Hk(i, k) + sn[i] * Hk(i + 1, k);
        Hk(i + 1, k) = -sn[i] * Hk(i, k) + cs[i] * Hk(i + 1, k);
        Hk(i, k) = t;
      }
      const double den = std::hypot(Hk(k, k), Hk(k + 1, k));
      cs[k] = den == 0.0 ? 1.0 : Hk(k, k) / den;
      sn[k] = den == 0.0 ? 0.0 : Hk(k + 1, k) / den;
      Hk(k, k) = den;
      Hk(k + 1, k) = 0.0;
      g[k + 1] = -sn[k] * g[k];
      g[k] = cs[k] * g[k];
      ++total;
      const double rel = std::abs(g[k + 1]) / rhs_norm;
      if (hist && hlen < hist_cap) hist[hlen] = rel;
      ++hlen;
      if (rel < tol || h_next == 0.0) done = true;
    }
    // back substitution, iterate update
    std::vector<double> y(k, 0.0);
    for (int i = k - 1; i >= 0; --i) {
      double acc = g[i];
      for (int j = i + 1; j < k; ++j) acc -= Hk(i, j) * y[j];
      y[i] = acc / Hk(i, i);
    }
    for (int j = 0; j < k; ++j)
      launch_axpy(x.get(), basis.get() + static_cast<std::int64_t>(j) * n, n, nullptr, 0.0, y[j], s);
    op(x.get(), w.get());
    launch_sub(r.get(), f.get(), w.get(), n, s);
    relres = norm_host(r.get()) / rhs_norm;
    if (relres < tol) converged = true;
  }
  H3D_CUDA_CHECK(cudaMemcpyAsync(xout, x.get(), n * 8, host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, s));
  end_call(s);
  H3D_CUDA_CHECK(cudaStreamSynchronize(s));
  if (info) {
    info->iterations = total;
    info->converged = converged ? 1 : 0;
    info->history_len = hlen;
    info->reserved = 0;
    info->solve_ms = ms_since(t0);
    info->final_relres = relres;
  }
}

}  // namespace h3db
