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

 private:
  T* p_ = nullptr;
  std::size_t n_ = 0;
};

struct LevelLists {
  // CSR per kind: 0 inter, 1 near_edge, 2 near_face
  std::vector<std::int32_t> off[3];
  std::vector<std::int32_t> ids[3];
};

struct LevelPairs {
  std::vector<std::int32_t> X, Y;      // Morton ids, X < Y
  std::vector<std::int32_t> rank;
  int threads = 32;                    // ACA CTA size (fixed per level: determinism)
  int max_m = 0, max_n = 0, max_mn = 0;
};

class Engine {
 public:
  Engine(const double* xyz, std::int64_t n, const h3d_options& opt);
  ~Engine();

  void matvec(const double* x, double* b, bool host, h3d_timing* t);
  void matvec_async(const double* x, double* b, cudaStream_t s);
  void profile(int enable, std::int64_t capacity);
  void profile_read(h3d_timing* sum, std::int64_t* steps);
  void stats(h3d_stats* out) const;
  void export_tree(std::int32_t* perm, int level, std::int64_t* offsets) const;
  std::int64_t export_list(int level, int kind, std::int32_t* offsets, std::int32_t* ids) const;
  std::int64_t export_pairs(int level, std::int32_t* x, std::int32_t* y, std::int32_t* rank) const;
  void attach_nccl(const void* id128, int rank, int world);

  std::mutex mu;  // serialises calls per handle (the handle owns stream + scratch)

 private:
  void build_tree(const double* xyz);
  void build_lists();
  void build_pairs();
  void run_aca(bool write);
  void build_layout();
  void build_matvec_plan();
  void near_scan();
  void check_flags(const char* where);
  std::int64_t enqueue(const double* xin, double* bout, cudaStream_t s, cudaEvent_t* ev);
  bool owned(int level, std::int64_t m) const;
  std::int64_t gid(int level, std::int64_t m) const { return node_base_[level] + m; }
  std::int64_t node_size(int level, std::int64_t m) const {
    return off_[level][m + 1] - off_[level][m];
  }

  h3d_options opt_;
  std::int64_t n_ = 0;
  int L_ = 0;
  int sms_ = 148;
  cudaStream_t stream_ = nullptr;
  cudaEvent_t ev_[8] = {};

  // tree
  std::vector<std::vector<std::int64_t>> off_;   // host offsets per level (8^l + 1)
  std::vector<std::int64_t> node_base_;          // global node id base per level
  std::int64_t total_nodes_ = 0;
  std::vector<std::int32_t> perm_h_;
  DevBuf<std::int32_t> perm_;
  DevBuf<double> px_, py_, pz_;
  DevBuf<std::int64_t> leaf_off_;
  DevBuf<unsigned> flags_;

  // ownership (Morton-subtree shard)
  int oct0_ = 0, oct1_ = 8;
  std::int64_t row0_ = 0, row1_ = 0;

  // lists / pairs
  std::vector<LevelLists> lists_;
  std::vector<LevelPairs> pairs_;
  // per level, per inter-list entry: pair index (-1 if not compressed here)
  std::vector<std::vector<std::int32_t>> entry_pair_;
  // per level, per inter-list entry: column offset of that partner in W_Z (-1: absent)
  std::vector<std::vector<std::int32_t>> entry_col_;

  // node tables (global ids)
  std::vector<std::int64_t> woff_h_, soff_h_, rowbeg_h_;
  std::vector<std::int32_t> rpad_h_, rows_h_;
  DevBuf<std::int64_t> woff_, soff_, rowbeg_;
  DevBuf<std::int32_t> rpad_, rows_;

  // pools
  DevBuf<double> W_, S_, P_;
  DevBuf<std::int32_t> spos_;
  std::int64_t w_doubles_ = 0, s_doubles_ = 0, p_doubles_ = 0;
  std::int64_t factor_doubles_ = 0, sum_rank_ = 0, npairs_ = 0, nblocks_ordered_ = 0;
  int max_rank_ = 0;
  std::uint64_t ref_float_count_ = 0, ref_int_count_ = 0;

  // matvec plan
  DevBuf<P1Item> p1_items_;
  DevBuf<P1Reduce> p1_red_;
  std::int64_t n_p1_ = 0, n_red_ = 0;
  DevBuf<std::int32_t> near_off_, near_ids_;
  DevBuf<std::int64_t> nf_off_;
  DevBuf<double> NF_;
  std::int64_t near_blocks_ = 0, near_entries_ = 0;
  std::int64_t leaf0_ = 0, leaf1_ = 0;  // owned leaves

  // matvec scratch
  DevBuf<double> x_, xp_, b_;

  // multi-GPU
  void* nccl_comm_ = nullptr;
  int world_ = 1, rank_ = 0;
  std::vector<std::int64_t> rank_row0_, rank_row1_;
  DevBuf<double> bperm_;

  // profiling ring for async matvecs (4 events per step)
  bool prof_on_ = false;
  std::vector<cudaEvent_t> prof_ev_;
  std::size_t prof_used_ = 0;
  std::int64_t prof_launches_ = 0;

  // timings
  double ms_tree_ = 0, ms_lists_ = 0, ms_aca_rank_ = 0, ms_aca_write_ = 0, ms_total_ = 0;
};

}  // namespace h3db
