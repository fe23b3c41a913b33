// Host orchestration: build (tree -> lists -> pairs -> ACA rank pass ->
// layout -> ACA write pass -> matvec plan) and the matvec launch sequence.
//
// Reference mapping:
//   Engine::Engine      <- h3d::initialize (hmatrix.cpp:52-151)
//   Engine::matvec      <- h3d::matvec (hmatrix.cpp:153-226); with shard_world > 1
//                          <- h3d::parallel_matvec (parallel.cpp:111-306)
//   Engine::stats       <- h3d::stats (hmatrix.cpp:228-251)
#include "engine.h"
#include "common.cuh"

#include <algorithm>
#include <chrono>
#include <cstring>
#include <numeric>

#include <nccl.h>

namespace h3db {

namespace {

using Clock = std::chrono::steady_clock;
double ms_since(Clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}

constexpr int kMaxDepth = 8;            // 8^8 leaves; beyond that the device tables explode
constexpr std::int64_t kRowChunk = 2048;  // phase-1 row chunk for tall nodes
constexpr int kColChunk = 256;          // phase-1 columns per item

#define NCCL_CHECK(expr)                                                        \
  do {                                                                          \
    ncclResult_t r_ = (expr);                                                   \
    if (r_ != ncclSuccess)                                                      \
      throw NcclFailure(std::string("NCCL error: ") + ncclGetErrorString(r_) + \
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
  world_ = opt.shard_world < 1 ? 1 : opt.shard_world;
  rank_ = opt.shard_rank;
  if (!(world_ == 1 || world_ == 2 || world_ == 4 || world_ == 8))
    throw InvalidArgument("initialize: shard_world must be 1, 2, 4 or 8 (Morton-subtree ownership)");
  if (rank_ < 0 || rank_ >= world_) throw InvalidArgument("initialize: shard_rank out of range");
  oct0_ = 8 * rank_ / world_;
  oct1_ = 8 * (rank_ + 1) / world_;

  H3D_CUDA_CHECK(cudaSetDevice(opt.device));
  cudaDeviceProp prop{};
  H3D_CUDA_CHECK(cudaGetDeviceProperties(&prop, opt.device));
  sms_ = prop.multiProcessorCount;
  H3D_CUDA_CHECK(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
  for (auto& e : ev_) H3D_CUDA_CHECK(cudaEventCreate(&e));

  auto t = Clock::now();
  build_tree(xyz);
  ms_tree_ = ms_since(t);
  t = Clock::now();
  build_lists();
  ms_lists_ = ms_since(t);
  build_pairs();
  t = Clock::now();
  run_aca(false);
  ms_aca_rank_ = ms_since(t);
  build_layout();
  t = Clock::now();
  run_aca(true);
  ms_aca_write_ = ms_since(t);
  build_matvec_plan();
  near_scan();
  H3D_CUDA_CHECK(cudaStreamSynchronize(stream_));
  ms_total_ = ms_since(t0);
}

Engine::~Engine() {
  for (auto e : prof_ev_)
    if (e) cudaEventDestroy(e);
  if (nccl_comm_) ncclCommDestroy(static_cast<ncclComm_t>(nccl_comm_));
  for (auto& e : ev_)
    if (e) cudaEventDestroy(e);
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

bool Engine::owned(int level, std::int64_t m) const {
  if (level == 0) return rank_ == 0;
  const std::int64_t oct = m >> (3 * (level - 1));
  return oct >= oct0_ && oct < oct1_;
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
  node_base_.assign(L_ + 2, 0);
  for (int l = 0; l <= L_; ++l) {
    const std::int64_t cnt = 1LL << (3 * l);
    DevBuf<std::int64_t> o;
    o.alloc(cnt + 1);
    launch_node_offsets(codes_s.get(), n_, cap, l, o.get(), stream_);
    off_[l].resize(cnt + 1);
    H3D_CUDA_CHECK(cudaMemcpyAsync(off_[l].data(), o.get(), (cnt + 1) * 8, cudaMemcpyDeviceToHost, stream_));
    H3D_CUDA_CHECK(cudaStreamSynchronize(stream_));
    node_base_[l + 1] = node_base_[l] + cnt;
  }
  total_nodes_ = node_base_[L_ + 1];
  perm_h_.resize(n_);
  H3D_CUDA_CHECK(cudaMemcpyAsync(perm_h_.data(), perm_.get(), n_ * 4, cudaMemcpyDeviceToHost, stream_));
  px_.alloc(n_);
  py_.alloc(n_);
  pz_.alloc(n_);
  launch_permute_points(xyz_d.get(), perm_.get(), n_, px_.get(), py_.get(), pz_.get(), stream_);
  leaf_off_.upload(off_[L_], stream_);
  H3D_CUDA_CHECK(cudaStreamSynchronize(stream_));
  // owned row range (Morton-subtree shard)
  if (L_ == 0) {
    row0_ = 0;
    row1_ = rank_ == 0 ? n_ : 0;
  } else {
    row0_ = off_[1][oct0_];
    row1_ = off_[1][oct1_];
  }
  rank_row0_.resize(world_);
  rank_row1_.resize(world_);
  for (int r = 0; r < world_; ++r) {
    if (L_ == 0) {
      rank_row0_[r] = 0;
      rank_row1_[r] = r == 0 ? n_ : 0;
    } else {
      rank_row0_[r] = off_[1][8 * r / world_];
      rank_row1_[r] = off_[1][8 * (r + 1) / world_];
    }
  }
}

// ---------------------------------------------------------------- lists
void Engine::build_lists() {
  lists_.assign(L_ + 1, LevelLists{});
  for (int k = 0; k < 3; ++k) lists_[0].off[k].assign(2, 0);
  if (L_ == 0) return;
  const std::int64_t maxcnt = 1LL << (3 * L_);
  const std::size_t tb = scan_temp_bytes(maxcnt);
  DevBuf<unsigned char> tmp;
  tmp.alloc(tb);
  DevBuf<std::int32_t> counts, offs;
  counts.alloc(3 * (maxcnt + 1));
  offs.alloc(3 * (maxcnt + 1));
  for (int l = 1; l <= L_; ++l) {
    const std::int64_t cnt = 1LL << (3 * l);
    H3D_CUDA_CHECK(cudaMemsetAsync(counts.get(), 0, 3 * (cnt + 1) * 4, stream_));
    launch_list_counts(l, counts.get(), stream_);
    for (int k = 0; k < 3; ++k)
      exclusive_scan_i32(tmp.get(), tb, counts.get() + k * (cnt + 1), offs.get() + k * (cnt + 1), cnt,
                         stream_);
    std::vector<std::int32_t> hoff(3 * (cnt + 1));
    H3D_CUDA_CHECK(cudaMemcpyAsync(hoff.data(), offs.get(), hoff.size() * 4, cudaMemcpyDeviceToHost, stream_));
    H3D_CUDA_CHECK(cudaStreamSynchronize(stream_));
    DevBuf<std::int32_t> ids[3];
    for (int k = 0; k < 3; ++k) {
      lists_[l].off[k].assign(hoff.begin() + k * (cnt + 1), hoff.begin() + (k + 1) * (cnt + 1));
      ids[k].alloc(lists_[l].off[k][cnt]);
    }
    launch_list_fill(l, offs.get(), ids[0].get(), ids[1].get(), ids[2].get(), stream_);
    for (int k = 0; k < 3; ++k) {
      lists_[l].ids[k].resize(lists_[l].off[k][cnt]);
      if (!lists_[l].ids[k].empty())
        H3D_CUDA_CHECK(cudaMemcpyAsync(lists_[l].ids[k].data(), ids[k].get(),
                                       lists_[l].ids[k].size() * 4, cudaMemcpyDeviceToHost, stream_));
    }
    H3D_CUDA_CHECK(cudaStreamSynchronize(stream_));
  }
}

// ---------------------------------------------------------------- pairs
// Admissible blocks (hmatrix.cpp:74-98) with both nodes non-empty; one ACA
// per unordered pair X < Y (the lists are swap-symmetric, octree tests
// test_octree.cpp:167-181, and the built-in kernels are symmetric,
// kernel.cpp:7-21). A shard compresses every pair touching an owned node.
void Engine::build_pairs() {
  pairs_.assign(L_ + 1, LevelPairs{});
  entry_pair_.assign(L_ + 1, {});
  entry_col_.assign(L_ + 1, {});
  nblocks_ordered_ = 0;
  for (int l = 1; l <= L_; ++l) {
    const std::int64_t cnt = 1LL << (3 * l);
    const auto& off = lists_[l].off[0];
    const auto& ids = lists_[l].ids[0];
    auto& ep = entry_pair_[l];
    ep.assign(ids.size(), -1);
    auto& P = pairs_[l];
    for (std::int64_t X = 0; X < cnt; ++X) {
      if (node_size(l, X) == 0) continue;
      for (std::int32_t e = off[X]; e < off[X + 1]; ++e) {
        const std::int32_t Y = ids[e];
        if (node_size(l, Y) == 0) continue;
        ++nblocks_ordered_;
        if (Y <= X || !(owned(l, X) || owned(l, Y))) continue;
        ep[e] = static_cast<std::int32_t>(P.X.size());
        P.X.push_back(static_cast<std::int32_t>(X));
        P.Y.push_back(Y);
        const int m = static_cast<int>(node_size(l, X)), nn = static_cast<int>(node_size(l, Y));
        P.max_m = std::max(P.max_m, m);
        P.max_n = std::max(P.max_n, nn);
        P.max_mn = std::max(P.max_mn, std::min(m, nn));
      }
    }
    for (std::int64_t Z = 0; Z < cnt; ++Z) {
      if (node_size(l, Z) == 0) continue;
      for (std::int32_t e = off[Z]; e < off[Z + 1]; ++e) {
        const std::int32_t k = ids[e];
        if (k >= Z || node_size(l, k) == 0 || !(owned(l, Z) || owned(l, k))) continue;
        // Z's position in k's sorted list
        const auto b = ids.begin() + off[k], en = ids.begin() + off[k + 1];
        const auto it = std::lower_bound(b, en, static_cast<std::int32_t>(Z));
        if (it == en || *it != Z) throw std::logic_error("interaction lists not swap-symmetric");
        ep[e] = ep[static_cast<std::size_t>(it - ids.begin())];
      }
    }
    P.rank.assign(P.X.size(), 0);
    const double mbar = static_cast<double>(n_) / static_cast<double>(cnt);
    P.threads = mbar <= 64 ? 32 : mbar <= 512 ? 128 : mbar <= 4096 ? 256 : 512;
  }
  npairs_ = 0;
  for (const auto& P : pairs_) npairs_ += static_cast<std::int64_t>(P.X.size());
}

// ---------------------------------------------------------------- ACA
void Engine::run_aca(bool write) {
  DevBuf<unsigned long long> counter;
  counter.alloc(1);
  std::size_t free_b = 0, total_b = 0;
  H3D_CUDA_CHECK(cudaMemGetInfo(&free_b, &total_b));
  for (int l = 1; l <= L_; ++l) {
    auto& P = pairs_[l];
    const std::int64_t np = static_cast<std::int64_t>(P.X.size());
    if (np == 0) continue;
    std::vector<std::int64_t> xb(np), yb(np), wx, wy;
    std::vector<std::int32_t> m(np), nn(np), rx, ry;
    for (std::int64_t p = 0; p < np; ++p) {
      xb[p] = off_[l][P.X[p]];
      yb[p] = off_[l][P.Y[p]];
      m[p] = static_cast<std::int32_t>(node_size(l, P.X[p]));
      nn[p] = static_cast<std::int32_t>(node_size(l, P.Y[p]));
    }
    DevBuf<std::int64_t> d_xb, d_yb, d_wx, d_wy;
    DevBuf<std::int32_t> d_m, d_n, d_rank, d_rx, d_ry;
    d_xb.upload(xb, stream_);
    d_yb.upload(yb, stream_);
    d_m.upload(m, stream_);
    d_n.upload(nn, stream_);
    d_rank.alloc(np);
    int level_max_rank = 0;
    if (write) {
      wx.resize(np);
      wy.resize(np);
      rx.resize(np);
      ry.resize(np);
      // column offsets of the pair in W_X and W_Y (build_layout)
      const auto& off = lists_[l].off[0];
      const auto& ids = lists_[l].ids[0];
      const auto& ec = entry_col_[l];
      for (std::int64_t p = 0; p < np; ++p) {
        const std::int32_t X = P.X[p], Y = P.Y[p];
        auto find = [&](std::int32_t a, std::int32_t b) {
          const auto it = std::lower_bound(ids.begin() + off[a], ids.begin() + off[a + 1], b);
          return static_cast<std::size_t>(it - ids.begin());
        };
        const std::int64_t gx = gid(l, X), gy = gid(l, Y);
        wx[p] = woff_h_[gx] + ec[find(X, Y)];
        rx[p] = rpad_h_[gx];
        wy[p] = woff_h_[gy] + ec[find(Y, X)];
        ry[p] = rpad_h_[gy];
        level_max_rank = std::max(level_max_rank, P.rank[p]);
      }
      d_wx.upload(wx, stream_);
      d_wy.upload(wy, stream_);
      d_rx.upload(rx, stream_);
      d_ry.upload(ry, stream_);
    }
    const int ms = (P.max_m + 1) & ~1, ns = (P.max_n + 1) & ~1;
    int cap_ws;
    if (write) {
      cap_ws = std::max(1, level_max_rank);
    } else {
      cap_ws = std::min(P.max_mn, P.threads == 32 ? 64 : 256);
      if (opt_.max_rank > 0) cap_ws = static_cast<int>(std::min<std::int64_t>(cap_ws, opt_.max_rank));
      cap_ws = std::max(cap_ws, 1);
    }
    for (;;) {
      const std::int64_t slot_doubles =
          static_cast<std::int64_t>(cap_ws + 1) * (ms + ns) + (ms + ns + 7) / 8 + 2;
      const std::size_t smem = aca_smem_bytes(P.threads, cap_ws);
      const int bps = aca_blocks_per_sm(P.threads, opt_.kernel_id, smem);
      const std::int64_t budget = std::max<std::int64_t>(
          std::min<std::int64_t>(static_cast<std::int64_t>(free_b / 4), 24LL << 30), 256LL << 20);
      std::int64_t slots = std::min<std::int64_t>(np, static_cast<std::int64_t>(bps) * sms_);
      slots = std::min<std::int64_t>(slots, std::max<std::int64_t>(1, budget / (slot_doubles * 8)));
      DevBuf<double> ws;
      ws.alloc(static_cast<std::size_t>(slots * slot_doubles));
      H3D_CUDA_CHECK(cudaMemsetAsync(counter.get(), 0, 8, stream_));
      H3D_CUDA_CHECK(cudaMemsetAsync(flags_.get(), 0, 4, stream_));
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
      a.ws = ws.get();
      a.slot_doubles = slot_doubles;
      a.cap_ws = cap_ws;
      a.ms = ms;
      a.ns = ns;
      a.rank_out = d_rank.get();
      if (write) {
        a.W = W_.get();
        a.wx = d_wx.get();
        a.rx = d_rx.get();
        a.wy = d_wy.get();
        a.ry = d_ry.get();
      }
      a.flags = flags_.get();
      a.counter = counter.get();
      launch_aca(a, P.threads, static_cast<int>(slots), stream_);
      unsigned f = 0;
      H3D_CUDA_CHECK(cudaMemcpyAsync(&f, flags_.get(), 4, cudaMemcpyDeviceToHost, stream_));
      H3D_CUDA_CHECK(cudaStreamSynchronize(stream_));
      if (f & kFlagDegenGeom) throw DegenerateGeometry("coincident distinct points in block");
      if (f & kFlagAcaOverflow) {
        if (write || cap_ws >= P.max_mn)
          throw std::logic_error("ACA workspace overflow in the write pass");
        cap_ws = std::min(2 * cap_ws, P.max_mn);
        continue;
      }
      break;
    }
    std::vector<std::int32_t> rk(np);
    H3D_CUDA_CHECK(cudaMemcpyAsync(rk.data(), d_rank.get(), np * 4, cudaMemcpyDeviceToHost, stream_));
    H3D_CUDA_CHECK(cudaStreamSynchronize(stream_));
    if (write) {
      if (rk != P.rank) throw std::logic_error("ACA write pass diverged from the rank pass");
    } else {
      P.rank = std::move(rk);
    }
  }
}

// ---------------------------------------------------------------- layout
// W_Z = [F_Z^(Z,k1) | F_Z^(Z,k2) | ...] over Z's partners in list order,
// row-major |Z| x rpad_Z (rpad even: 16-byte rows). S shares the column
// layout; spos maps a column of W_Z to the S slot of the mirrored block.
void Engine::build_layout() {
  woff_h_.assign(total_nodes_, 0);
  soff_h_.assign(total_nodes_, 0);
  rowbeg_h_.assign(total_nodes_, 0);
  rpad_h_.assign(total_nodes_, 0);
  rows_h_.assign(total_nodes_, 0);
  for (int l = 0; l <= L_; ++l) {
    const std::int64_t cnt = 1LL << (3 * l);
    for (std::int64_t z = 0; z < cnt; ++z) {
      rowbeg_h_[gid(l, z)] = off_[l][z];
      rows_h_[gid(l, z)] = static_cast<std::int32_t>(node_size(l, z));
    }
  }
  std::int64_t wtot = 0, stot = 0;
  factor_doubles_ = sum_rank_ = 0;
  max_rank_ = 0;
  ref_float_count_ = ref_int_count_ = 0;
  for (int l = 1; l <= L_; ++l) {
    const auto& P = pairs_[l];
    for (std::size_t p = 0; p < P.X.size(); ++p) {
      const std::int64_t r = P.rank[p];
      sum_rank_ += r;
      factor_doubles_ += r * (node_size(l, P.X[p]) + node_size(l, P.Y[p]));
      max_rank_ = std::max(max_rank_, P.rank[p]);
      ref_float_count_ += 2ull * static_cast<std::uint64_t>(r * r);
      ref_int_count_ += 4ull * static_cast<std::uint64_t>(r);
    }
    const std::int64_t cnt = 1LL << (3 * l);
    const auto& off = lists_[l].off[0];
    const auto& ep = entry_pair_[l];
    auto& ec = entry_col_[l];
    ec.assign(ep.size(), -1);
    for (std::int64_t z = 0; z < cnt; ++z) {
      std::int32_t cols = 0;
      bool any = false;
      for (std::int32_t e = off[z]; e < off[z + 1]; ++e) {
        if (ep[e] < 0) continue;
        ec[e] = cols;
        cols += P.rank[ep[e]];
        any = true;
      }
      const std::int64_t g = gid(l, z);
      const std::int32_t rpad = any ? cols + (cols & 1) : 0;
      rpad_h_[g] = rpad;
      woff_h_[g] = wtot;
      soff_h_[g] = stot;
      wtot += node_size(l, z) * rpad;
      stot += rpad;
    }
  }
  w_doubles_ = wtot;
  s_doubles_ = stot;
  if (stot > 0x7fffffffLL) throw InvalidArgument("initialize: t-vector pool exceeds int32 indexing");
  std::vector<std::int32_t> spos(std::max<std::int64_t>(stot, 1), -1);
  for (int l = 1; l <= L_; ++l) {
    const std::int64_t cnt = 1LL << (3 * l);
    const auto& off = lists_[l].off[0];
    const auto& ids = lists_[l].ids[0];
    const auto& ep = entry_pair_[l];
    const auto& ec = entry_col_[l];
    const auto& P = pairs_[l];
    for (std::int64_t z = 0; z < cnt; ++z) {
      for (std::int32_t e = off[z]; e < off[z + 1]; ++e) {
        if (ep[e] < 0) continue;
        const std::int32_t k = ids[e];
        if (!owned(l, k)) continue;  // only owned targets run phase 2
        const int r = P.rank[ep[e]];
        const auto it = std::lower_bound(ids.begin() + off[k], ids.begin() + off[k + 1],
                                         static_cast<std::int32_t>(z));
        const std::int32_t e2 = ec[static_cast<std::size_t>(it - ids.begin())];
        const std::int64_t src = soff_h_[gid(l, z)] + ec[e];
        const std::int64_t dst = soff_h_[gid(l, k)] + e2;
        for (int a = 0; a < r; ++a) spos[src + a] = static_cast<std::int32_t>(dst + a);
      }
    }
  }
  W_.alloc(std::max<std::int64_t>(wtot, 2));
  H3D_CUDA_CHECK(cudaMemsetAsync(W_.get(), 0, W_.size() * 8, stream_));
  S_.alloc(std::max<std::int64_t>(stot, 2));
  H3D_CUDA_CHECK(cudaMemsetAsync(S_.get(), 0, S_.size() * 8, stream_));
  spos_.upload(spos, stream_);
  woff_.upload(woff_h_, stream_);
  soff_.upload(soff_h_, stream_);
  rowbeg_.upload(rowbeg_h_, stream_);
  rpad_.upload(rpad_h_, stream_);
  rows_.upload(rows_h_, stream_);
  H3D_CUDA_CHECK(cudaStreamSynchronize(stream_));
}

// ---------------------------------------------------------------- plan
void Engine::build_matvec_plan() {
  std::vector<P1Item> items;
  std::vector<P1Reduce> reds;
  std::int64_t ptot = 0;
  for (int l = 1; l <= L_; ++l) {
    const std::int64_t cnt = 1LL << (3 * l);
    for (std::int64_t z = 0; z < cnt; ++z) {
      const std::int64_t g = gid(l, z);
      const int rpad = rpad_h_[g];
      if (rpad == 0) continue;
      const std::int64_t rows = node_size(l, z);
      const std::int64_t nrc = (rows + kRowChunk - 1) / kRowChunk;
      const int ncc = (rpad + kColChunk - 1) / kColChunk;
      const std::int64_t pbase = ptot;
      if (nrc > 1) {
        ptot += nrc * rpad;
        reds.push_back(P1Reduce{static_cast<std::int32_t>(g), rpad, static_cast<std::int32_t>(nrc), 0, pbase});
      }
      for (std::int64_t k = 0; k < nrc; ++k)
        for (int cc = 0; cc < ncc; ++cc) {
          P1Item it{};
          it.node = static_cast<std::int32_t>(g);
          it.row0 = static_cast<std::int32_t>(k * kRowChunk);
          it.nrows = static_cast<std::int32_t>(std::min<std::int64_t>(kRowChunk, rows - k * kRowChunk));
          it.col0 = cc * kColChunk;
          it.ncols = std::min(kColChunk, rpad - cc * kColChunk);
          it.pslot = nrc > 1 ? pbase + k * rpad + cc * kColChunk : -1;
          items.push_back(it);
        }
    }
  }
  n_p1_ = static_cast<std::int64_t>(items.size());
  n_red_ = static_cast<std::int64_t>(reds.size());
  p_doubles_ = ptot;
  p1_items_.upload(items, stream_);
  p1_red_.upload(reds, stream_);
  P_.alloc(std::max<std::int64_t>(ptot, 1));

  // leaf near lists: self, near_edge, near_face (non-empty), visit order of
  // the reference dense pass (hmatrix.cpp:105-120)
  const std::int64_t nl = 1LL << (3 * L_);
  if (L_ == 0) {
    leaf0_ = 0;
    leaf1_ = rank_ == 0 ? 1 : 0;
  } else {
    leaf0_ = static_cast<std::int64_t>(oct0_) << (3 * (L_ - 1));
    leaf1_ = static_cast<std::int64_t>(oct1_) << (3 * (L_ - 1));
  }
  std::vector<std::int32_t> noff(nl + 1, 0), nids;
  std::vector<std::int64_t> nfoff(nl + 1, 0);
  std::int64_t nftot = 0;
  near_blocks_ = near_entries_ = 0;
  for (std::int64_t x = 0; x < nl; ++x) {
    noff[x] = static_cast<std::int32_t>(nids.size());
    nfoff[x] = nftot;
    const std::int64_t mx = node_size(L_, x);
    if (mx == 0 || x < leaf0_ || x >= leaf1_) continue;
    std::int64_t ntot = 0;
    auto add = [&](std::int64_t y) {
      const std::int64_t ny = node_size(L_, y);
      if (ny == 0) return;
      nids.push_back(static_cast<std::int32_t>(y));
      ntot += ny;
      ++near_blocks_;
      near_entries_ += mx * ny;
    };
    add(x);
    if (L_ > 0)
      for (int k = 1; k <= 2; ++k)
        for (std::int32_t e = lists_[L_].off[k][x]; e < lists_[L_].off[k][x + 1]; ++e)
          add(lists_[L_].ids[k][e]);
    nftot += mx * ntot;
  }
  noff[nl] = static_cast<std::int32_t>(nids.size());
  nfoff[nl] = nftot;
  near_off_.upload(noff, stream_);
  near_ids_.upload(nids.empty() ? std::vector<std::int32_t>{0} : nids, stream_);
  if (opt_.near_mode == H3D_NEAR_STORED) {
    nf_off_.upload(nfoff, stream_);
    NF_.alloc(std::max<std::int64_t>(nftot, 1));
  }
  x_.alloc(n_);
  xp_.alloc(n_);
  b_.alloc(n_);
  H3D_CUDA_CHECK(cudaStreamSynchronize(stream_));
}

void Engine::near_scan() {
  if (leaf1_ <= leaf0_) return;
  Phase2Args a;
  a.depth = L_;
  a.leaf0 = leaf0_;
  a.nleaves = leaf1_ - leaf0_;
  a.leaf_off = leaf_off_.get();
  a.px = px_.get();
  a.py = py_.get();
  a.pz = pz_.get();
  a.near_off = near_off_.get();
  a.near_ids = near_ids_.get();
  a.nf_off = opt_.near_mode == H3D_NEAR_STORED ? nf_off_.get() : nullptr;
  a.kernel = opt_.kernel_id;
  a.diag = opt_.diagonal;
  H3D_CUDA_CHECK(cudaMemsetAsync(flags_.get(), 0, 4, stream_));
  launch_near_scan(a, opt_.near_mode == H3D_NEAR_STORED ? NF_.get() : nullptr, flags_.get(), stream_);
  check_flags("near field");
}

// ---------------------------------------------------------------- matvec
// Enqueue one matvec on stream s: x (original order, device) -> b (original
// order, device). ev (optional, 4 events) brackets gather/exchange, phase 1,
// phase 2. Returns the number of kernels launched.
std::int64_t Engine::enqueue(const double* xin, double* bout, cudaStream_t s, cudaEvent_t* ev) {
  std::int64_t launches = 0;
  if (ev) cudaEventRecord(ev[0], s);
  if (world_ == 1) {
    launch_gather(xin, perm_.get(), n_, xp_.get(), s);
    ++launches;
  } else {
    // own slice of x in Morton order, then the all-gather of x over NVLink
    if (row1_ > row0_) {
      launch_gather(xin, perm_.get() + row0_, row1_ - row0_, xp_.get() + row0_, s);
      ++launches;
    }
    auto comm = static_cast<ncclComm_t>(nccl_comm_);
    NCCL_CHECK(ncclGroupStart());
    for (int r = 0; r < world_; ++r) {
      const std::int64_t c = rank_row1_[r] - rank_row0_[r];
      if (c > 0)
        NCCL_CHECK(ncclBroadcast(xp_.get() + rank_row0_[r], xp_.get() + rank_row0_[r],
                                 static_cast<std::size_t>(c), ncclDouble, r, comm, s));
    }
    NCCL_CHECK(ncclGroupEnd());
  }
  if (ev) cudaEventRecord(ev[1], s);
  NodeTable nt{rowbeg_.get(), rows_.get(), woff_.get(), rpad_.get(), soff_.get()};
  launch_phase1(p1_items_.get(), n_p1_, nt, W_.get(), xp_.get(), spos_.get(), S_.get(), P_.get(), s);
  launches += n_p1_ > 0;
  launch_phase1_reduce(p1_red_.get(), n_red_, nt, spos_.get(), P_.get(), S_.get(), s);
  launches += n_red_ > 0;
  if (ev) cudaEventRecord(ev[2], s);
  if (leaf1_ > leaf0_) {
    Phase2Args a;
    a.depth = L_;
    a.leaf0 = leaf0_;
    a.nleaves = leaf1_ - leaf0_;
    a.leaf_off = leaf_off_.get();
    a.nt = nt;
    a.W = W_.get();
    a.S = S_.get();
    a.xp = xp_.get();
    a.px = px_.get();
    a.py = py_.get();
    a.pz = pz_.get();
    a.perm = perm_.get();
    a.near_off = near_off_.get();
    a.near_ids = near_ids_.get();
    if (opt_.near_mode == H3D_NEAR_STORED) {
      a.nf_off = nf_off_.get();
      a.NF = NF_.get();
    }
    a.kernel = opt_.kernel_id;
    a.diag = opt_.diagonal;
    a.b = bout;
    for (int l = 0; l <= L_ && l < 24; ++l) a.lbase[l] = node_base_[l];
    launch_phase2(a, s);
    ++launches;
  }
  if (ev) cudaEventRecord(ev[3], s);
  return launches;
}

void Engine::matvec(const double* x, double* b, bool host, h3d_timing* t) {
  H3D_CUDA_CHECK(cudaSetDevice(opt_.device));
  if (world_ > 1 && nccl_comm_ == nullptr)
    throw InvalidArgument("matvec: sharded engine needs h3d_dev_attach_nccl first");
  cudaEventRecord(ev_[0], stream_);
  const double* xin = x;
  if (host) {
    H3D_CUDA_CHECK(cudaMemcpyAsync(x_.get(), x, n_ * 8, cudaMemcpyHostToDevice, stream_));
    xin = x_.get();
  }
  double* bout = host ? b_.get() : b;
  const std::int64_t launches = enqueue(xin, bout, stream_, ev_ + 1);
  if (host) H3D_CUDA_CHECK(cudaMemcpyAsync(b, b_.get(), n_ * 8, cudaMemcpyDeviceToHost, stream_));
  cudaEventRecord(ev_[5], stream_);
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
    if (world_ == 1) t->gather_ms = el(1, 2);
    else t->exchange_ms = el(1, 2);
    t->phase1_ms = el(2, 3);
    t->phase2_ms = el(3, 4);
    t->d2h_ms = el(4, 5);
    t->launches = launches;
  }
}

void Engine::matvec_async(const double* x, double* b, cudaStream_t s) {
  H3D_CUDA_CHECK(cudaSetDevice(opt_.device));
  if (world_ > 1 && nccl_comm_ == nullptr)
    throw InvalidArgument("matvec: sharded engine needs h3d_dev_attach_nccl first");
  cudaEvent_t* ev = nullptr;
  if (prof_on_) {
    if (prof_used_ >= prof_ev_.size() / 4) throw InvalidArgument("profile ring full; read it first");
    ev = prof_ev_.data() + 4 * prof_used_;
    ++prof_used_;
  }
  prof_launches_ += enqueue(x, b, s, ev);
}

void Engine::profile(int enable, std::int64_t capacity) {
  H3D_CUDA_CHECK(cudaSetDevice(opt_.device));
  prof_on_ = enable != 0;
  prof_used_ = 0;
  prof_launches_ = 0;
  const std::size_t need = static_cast<std::size_t>(4 * std::max<std::int64_t>(capacity, 1));
  if (prof_on_ && prof_ev_.size() < need) {
    for (auto e : prof_ev_) cudaEventDestroy(e);
    prof_ev_.assign(need, nullptr);
    for (auto& e : prof_ev_) H3D_CUDA_CHECK(cudaEventCreate(&e));
  }
}

void Engine::profile_read(h3d_timing* sum, std::int64_t* steps) {
  H3D_CUDA_CHECK(cudaSetDevice(opt_.device));
  std::memset(sum, 0, sizeof(*sum));
  for (std::size_t k = 0; k < prof_used_; ++k) {
    cudaEvent_t* ev = prof_ev_.data() + 4 * k;
    H3D_CUDA_CHECK(cudaEventSynchronize(ev[3]));
    float a = 0, b = 0, c = 0;
    cudaEventElapsedTime(&a, ev[0], ev[1]);
    cudaEventElapsedTime(&b, ev[1], ev[2]);
    cudaEventElapsedTime(&c, ev[2], ev[3]);
    if (world_ == 1) sum->gather_ms += a;
    else sum->exchange_ms += a;
    sum->phase1_ms += b;
    sum->phase2_ms += c;
    sum->total_ms += a + b + c;
  }
  sum->launches = prof_launches_;
  *steps = static_cast<std::int64_t>(prof_used_);
  prof_used_ = 0;
  prof_launches_ = 0;
}

void Engine::attach_nccl(const void* id128, int rank, int world) {
  if (world != world_ || rank != rank_)
    throw InvalidArgument("attach_nccl: rank/world differ from the engine's shard options");
  H3D_CUDA_CHECK(cudaSetDevice(opt_.device));
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  ncclComm_t comm;
  NCCL_CHECK(ncclCommInitRank(&comm, world, id, rank));
  nccl_comm_ = comm;
}

void Engine::stats(h3d_stats* s) const {
  std::memset(s, 0, sizeof(*s));
  s->depth = L_;
  s->max_rank = max_rank_;
  s->n = n_;
  s->lowrank_blocks = nblocks_ordered_;
  s->aca_pairs = npairs_;
  s->sum_rank = sum_rank_;
  s->factor_doubles = factor_doubles_;
  s->factor_bytes_alloc = w_doubles_ * 8;
  s->tvec_doubles = s_doubles_;
  s->near_blocks = near_blocks_;
  s->near_entries = near_entries_;
  s->near_bytes_stored = opt_.near_mode == H3D_NEAR_STORED ? near_entries_ * 8 : 0;
  s->ref_float_count = ref_float_count_ + static_cast<std::uint64_t>(near_entries_);
  s->ref_int_count = ref_int_count_;
  s->compression_ratio = static_cast<double>(s->ref_float_count) /
                         (static_cast<double>(n_) * static_cast<double>(n_));
  s->build_ms_tree = ms_tree_;
  s->build_ms_lists = ms_lists_;
  s->build_ms_aca_rank = ms_aca_rank_;
  s->build_ms_aca_write = ms_aca_write_;
  s->build_ms_total = ms_total_;
  s->phase1_items = n_p1_;
  s->owned_row_begin = row0_;
  s->owned_row_end = row1_;
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
  if (level < 0 || level > L_ || kind < 0 || kind > 2)
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
  const auto& P = pairs_[level];
  if (x) std::memcpy(x, P.X.data(), P.X.size() * 4);
  if (y) std::memcpy(y, P.Y.data(), P.Y.size() * 4);
  if (rank) std::memcpy(rank, P.rank.data(), P.rank.size() * 4);
  return static_cast<std::int64_t>(P.X.size());
}

}  // namespace h3db
