// Host orchestration of the B200 HODLR3D engine (C++; no torch types).
#pragma once

#include <cstdint>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/h3d_b200.h"
#include "kernels.h"
#include "planner.h"

namespace h3db {

// Exception types mirroring the reference's (kernel.hpp:64-66, octree.hpp:41-43).
struct InvalidArgument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct DegenerateGeometry : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct DegenerateDistribution : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NcclFailure : std::runtime_error {
  using std::runtime_error::runtime_error;
};

template <class T>
class DevBuf {
 public:
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { reset(); }
  void alloc(std::size_t n);
  void reset();
  T* get() const { return p_; }
  std::size_t size() const { return n_; }
  void upload(const T* h, std::size_t n, cudaStream_t s);
  void upload(const std::vector<T>& h, cudaStream_t s) { upload(h.data(), h.size(), s); }
  void swap(DevBuf& o) {
    std::swap(p_, o.p_);
    std::swap(n_, o.n_);
  }

 private:
  T* p_ = nullptr;
  std::size_t n_ = 0;
};

class Engine {
 public:
  Engine(const double* xyz, std::int64_t n, const h3d_options& opt);
  ~Engine();

  void matvec(const double* x, double* b, bool host, h3d_timing* t);
  void matvec_async(const double* x, double* b, cudaStream_t s);
  void profile(int enable, std::int64_t capacity);
  void profile_read(h3d_timing* sum, std::int64_t* steps);
  void profile_kernels(double* ms_sum, std::int64_t* launches, double* start_sum, int count) const;
  void stats(h3d_stats* out) const;
  void export_tree(std::int32_t* perm, int level, std::int64_t* offsets) const;
  std::int64_t export_list(int level, int kind, std::int32_t* offsets, std::int32_t* ids) const;
  std::int64_t export_pairs(int level, std::int32_t* x, std::int32_t* y, std::int32_t* rank) const;
  void attach_nccl(const void* id128, int rank, int world);
  void comm_ledger(h3d_comm_ledger* out) const;
  // exact dense product b = K x (O(N^2), verification / manufactured RHS)
  void direct_matvec(const double* x, double* b, bool host);
  // relative 2-norm error of b against exact row sums (reference
  // hmatrix.cpp:253-291): every row if N <= exact_limit, else sample_rows
  // Morton positions drawn by mt19937_64(seed)
  double reference_error(const double* x, const double* b, bool host, std::int64_t exact_limit,
                         std::int64_t sample_rows, std::uint64_t seed);
  // GMRES on (alpha I + beta A) x = rhs, reference solver.cpp:22-125
  void gmres(const double* rhs, double* x, bool host, double alpha, double beta, double tol, int restart,
             int max_iter, double* hist, int hist_cap, h3d_gmres_info* info);

  std::mutex mu;  // serialises calls per handle (the handle owns stream + scratch)

 private:
  void build_tree(const double* xyz);
  void build_lists();
  void run_aca(bool write);
  // single-pass build: the rank pass leaves every pair's pivots + packed LU in
  // a bump pool; afterwards proxy levels compact it into place and stream /
  // pair levels generate their explicit factors from it (factor_gen)
  bool finish_single_pass();
  DevBuf<double> pool_;
  DevBuf<unsigned long long> pool_ctr_;
  std::vector<std::unique_ptr<DevBuf<std::int64_t>>> pool_off_;  // per level
  bool pool_ok_ = false;
  void choose_modes();
  void upload_plan();
  void near_scan();
  void check_flags(const char* where);
  std::int64_t enqueue(const double* xin, double* bout, cudaStream_t s, cudaEvent_t* ev,
                       std::uint32_t* kmask);
  // Calls that use the handle's scratch (counters, S pool, partials, x in
  // Morton order) are ordered on the device: each waits for the previous
  // call's completion event when it runs on a different stream, and records
  // its own. Two matvec_async calls on different caller streams are then
  // serialised exactly like two calls on one stream (reference
  // hmatrix.hpp:34-36: the representation is shareable).
  void begin_call(cudaStream_t s);
  void end_call(cudaStream_t s);
  cudaEvent_t done_ev_ = nullptr;
  cudaStream_t last_stream_ = nullptr;
  bool done_valid_ = false;
  Phase2Args phase2_args(double* bout) const;
  std::int64_t node_size(int level, std::int64_t m) const {
    return off_[level][m + 1] - off_[level][m];
  }

  h3d_options opt_;
  std::int64_t n_ = 0;
  int L_ = 0;
  int sms_ = 148;
  // persistent-CTA residency per SM of the matvec kernels when the HBM and
  // FP64 lanes share the SMs; overridable for tuning through
  // H3D_TUNE="p1s=1,p1p=4,p2c=2,p2s=1,p2p=4" (proxy kernels: 128-thread CTAs)
  // ("skip=<mask of h3d_kernel_slot>" drops kernels: timing experiments only,
  // results are wrong; honoured only in a -DH3D_DEVTOOLS build)
  // ("nf=0": near field after p2_proxy instead of forked beside the solves,
  // "nf=1": forked right after p1_proxy, "nf=2": forked after the two-use
  // pass (the default when there is one, else 1);
  // "nfc": CTAs per SM of the forked near kernel; "fw=0": p2_stream does not
  // wait for the solves-done flag; "sol": CTAs per SM of the proxy solve;
  // "p2o=0": phase-2 FP64 kernels do not wait for the HBM lane's phase 1;
  // "acab": cap on the ACA CTAs per SM, 0 = occupancy limit; "acat<l>=<n>":
  // ACA CTA size of level l)
  struct Tune {
    int p1s = 1, p1p = 4, p2c = 2, p2s = 1, p2p = 4, skip = 0, h2w = 1, nf = -1, nfc = 1, pps = 0, graphs = 1, fw = 1,
        sol = 2, p2o = 1, acab = 0, half_search = 0, nfd = 0;
    int acat[16] = {};  // per-level ACA CTA size override (32 / 128 / 256 / 512)
  } tune_;
  std::size_t free_mem_ = 0;
  cudaStream_t stream_ = nullptr;
  cudaEvent_t ev_[8] = {};

  // tree (device) + host offsets / lists
  std::vector<std::vector<std::int64_t>> off_;
  std::vector<LevelLists> lists_;
  std::vector<std::int32_t> perm_h_;
  DevBuf<std::int32_t> perm_;
  DevBuf<double> px_, py_, pz_;
  DevBuf<double> p4_;  // packed (x, y, z, x-value) per permuted point
  DevBuf<std::int64_t> leaf_off_;
  DevBuf<unsigned> flags_;

  std::unique_ptr<Planner> plan_;
  std::vector<int> modes_;
  int world_ = 1, rank_ = 0;

  // device copies of the plan
  DevBuf<std::int64_t> woff_, soff_, rowbeg_;
  DevBuf<std::int32_t> rpad_, rows_;
  DevBuf<double> W_, S_, P_;
  DevBuf<std::int32_t> spos_;
  DevBuf<std::int32_t> piv_;
  DevBuf<double> lu_;
  std::int64_t lu_total_ = 0;
  DevBuf<double> q4_;  // proxy points (x, y, z, -) in S index space
  DevBuf<double> q4c_;  // the same points centred on their node's box (x', y', z', |.|^2)
  DevBuf<double> center_;  // box centre per global node
  DevBuf<std::int32_t> vcols_;  // leading vertex-partner columns per node
  DevBuf<ProxySeg> segs_all_, segs_solve_, segs_solve2_;
  // segs_solve2_: split levels' Y-role segments, solved before the two-use pass
  std::int64_t n_segs_all_ = 0, n_segs_solve_ = 0, n_segs_solve2_ = 0;
  DevBuf<P1Item> p1_stream_items_, p1_proxy_items_;
  DevBuf<P1Reduce> p1_red_s_, p1_red_p_, p1_red_h_;  // tall-node partial reductions, stream / proxy / half kind
  std::int64_t n_p1s_ = 0, n_p1p_ = 0, n_red_s_ = 0, n_red_p_ = 0, n_red_h_ = 0;
  DevBuf<H2Item> h2_items_;  // half levels, regenerated side (both uses per entry)
  std::int64_t n_h2_ = 0;
  cudaEvent_t h2_done_ = nullptr;  // the half pass's v are in S (p2_stream waits)
  bool has_stream_levels_ = false;
  DevBuf<std::int32_t> near_off_, near_ids_, near_dense_;
  DevBuf<std::int32_t> sym_off_, sym_ids_, sym_cnt_, in_off_;
  DevBuf<std::int64_t> out_off_, in_pos_;
  DevBuf<double> pairbuf_;  // symmetric near-field column sums (owned pairs)
  bool sym_near_ = false;   // near field with pair symmetry (always on; both near modes)
  DevBuf<double> cpart_;
  DevBuf<P2Item> p2_items_, p2s_items_;
  DevBuf<StreamDesc> p1s_desc_, p2s_desc_;
  DevBuf<PairDesc> pair_descs_;          // pair levels (kModePair)
  std::vector<std::int64_t> pd_level_;   // descriptor range per level
  DevBuf<FusedDesc> fused_descs_;        // fused levels (kModeFused)
  std::vector<std::int64_t> fd_level_, pg_level_;
  std::int64_t pg_pair_[2] = {0, 0}, pg_fused_[2] = {0, 0};  // gather item ranges per lane
  DevBuf<std::int32_t> pc_off_;
  DevBuf<std::int64_t> pc_pos_;
  DevBuf<P2Item> pg_items_;
  std::int64_t n_pg_ = 0;
  DevBuf<double> pair_out_;
  std::int64_t n_p2_ = 0, n_p2s_ = 0;
  int n_lvl_ = 0;
  DevBuf<double> lvl_part_;  // [n_lvl_ x N] phase-2 per-level partials
  DevBuf<unsigned> sync_flag_;  // solves done (FP64 lane -> HBM lane): reset per matvec, set to 1
  // CUDA graphs of the whole matvec (both lanes, fork/join), one per (x, b)
  // pair seen twice; replayed on the caller's stream
  struct GraphEntry {
    const double* x = nullptr;
    double* b = nullptr;
    cudaGraphExec_t exec = nullptr;
    std::int64_t launches = 0;
    int seen = 0;
  };
  std::vector<GraphEntry> graphs_;
  std::int64_t run_graph(const double* x, double* b, cudaStream_t s);
  // work counters: [p1_stream, p1_proxy, p2_compute, p2_stream, p2_proxy, solve, two-use pass, solve 2,
  // pair levels 8..]
  static constexpr int kCounters = 32;
  DevBuf<unsigned> counters_;
  // matvec lanes (priorities: the HBM lane and the FP64 critical chain above
  // the near field, which fills whatever the two leave idle)
  cudaStream_t stream2_ = nullptr;          // HBM lane: stream levels
  cudaStream_t stream3_ = nullptr;          // near field + direct leaf blocks (needs x only)
  cudaStream_t stream4_ = nullptr;          // FP64 lane: proxy levels + solves
  cudaEvent_t fork_[3] = {}, join_[3] = {};
  DevBuf<std::int64_t> nf_off_;
  DevBuf<std::int32_t> nf_cols_;
  DevBuf<double> NF_;

  // matvec scratch
  DevBuf<double> x_, xp_, b_;

  // multi-GPU
  void* nccl_comm_ = nullptr;
  DevBuf<double> bm_;           // Morton-order b for the all-gather (gather_b)
  bool force_gather_ = false;   // GMRES on a sharded handle: every matvec returns the full b
  std::int64_t comm_matvecs_ = 0;

  // profiling ring for async matvecs (4 events per step)
  bool prof_on_ = false;
  // per profiled call: 4 phase events + a (begin, end) pair per kernel slot
  static constexpr int kProfEv = 4 + 2 * H3D_K_COUNT;
  std::vector<cudaEvent_t> prof_ev_;
  std::vector<std::uint32_t> prof_mask_;  // kernel slots recorded per call
  double prof_kms_[H3D_K_COUNT] = {};
  double prof_kstart_[H3D_K_COUNT] = {};
  std::int64_t prof_kn_[H3D_K_COUNT] = {};
  std::size_t prof_used_ = 0;
  std::int64_t prof_launches_ = 0;

  // build timings
  double ms_tree_ = 0, ms_lists_ = 0, ms_aca_rank_ = 0, ms_aca_write_ = 0, ms_total_ = 0, ms_plan_ = 0,
         ms_post_ = 0, ms_near_ = 0;
  bool single_pass_ = false;  // the build skipped the ACA write pass
  double level_aca_ms_[16] = {};  // rank + write pass per level
};

}  // namespace h3db
