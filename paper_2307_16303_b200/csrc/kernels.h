// Launch interfaces of the sm_100a kernels (host-callable, no torch types).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>

#include <cuda_runtime.h>

#include "planner.h"

namespace h3db {

struct CudaError : std::runtime_error {
  CudaError(cudaError_t e, const char* expr, const char* file, int line)
      : std::runtime_error(std::string("CUDA error ") + cudaGetErrorString(e) + " at " + file +
                           ":" + std::to_string(line) + " (" + expr + ")"),
        code(e) {}
  cudaError_t code;
};

// ---------------------------------------------------------------- tree.cu
// Morton codes at depth_cap (reference octree.cpp:67-72, 99-108), fp64
// binning with round-to-nearest multiplies exactly as the reference.
void launch_morton_codes(const double* xyz, std::int64_t n, int depth_cap,
                         unsigned long long* codes, std::int32_t* idx, unsigned* flags,
                         cudaStream_t s);
std::size_t radix_sort_temp_bytes(std::int64_t n, int end_bit);
void radix_sort_pairs(void* tmp, std::size_t tmp_bytes, const unsigned long long* kin,
                      unsigned long long* kout, const std::int32_t* vin, std::int32_t* vout,
                      std::int64_t n, int end_bit, cudaStream_t s);
// max run length of (code >> 3(cap-l)) for every l in [0, cap] (octree.cpp:110-130)
void launch_depth_scan(const unsigned long long* codes, std::int64_t n, int depth_cap,
                       unsigned long long* maxocc, cudaStream_t s);
// node offsets at `level`: off[m] = first sorted index with prefix >= m, m in [0, 8^l]
void launch_node_offsets(const unsigned long long* codes, std::int64_t n, int depth_cap,
                         int level, std::int64_t* off, cudaStream_t s);
void launch_permute_points(const double* xyz, const std::int32_t* perm, std::int64_t n,
                           double* px, double* py, double* pz, cudaStream_t s);

// --------------------------------------------------------------- lists.cu
// Interaction lists at one level (octree.cpp:197-260) for a variant: kind 0
// inter, 1 near_edge, 2 near_face, 3 near_vertex. counts: kListKinds x (8^l + 1).
void launch_list_counts(int level, int variant, std::int32_t* counts, cudaStream_t s);
void launch_list_fill(int level, int variant, const std::int32_t* offsets, std::int32_t* const* ids,
                      cudaStream_t s);
// exclusive scan of n int32 into int32 (n+1 outputs, last = total)
std::size_t scan_temp_bytes(std::int64_t n);
void exclusive_scan_i32(void* tmp, std::size_t tmp_bytes, const std::int32_t* in,
                        std::int32_t* out, std::int64_t n, cudaStream_t s);

// ----------------------------------------------------------------- aca.cu
struct AcaArgs {
  std::int64_t npairs = 0;
  std::int64_t nclaims = -1;  // pairs this launch claims (order[0 .. nclaims)); < 0: npairs
  const std::int64_t* xb = nullptr;  // row range begin (permuted index)
  const std::int32_t* m = nullptr;
  const std::int64_t* yb = nullptr;  // column range begin
  const std::int32_t* n = nullptr;
  const double *px = nullptr, *py = nullptr, *pz = nullptr;
  int kernel = 0;
  double diag = 0.0;
  double eps = 1e-7;
  std::int64_t max_rank = 0;
  // workspace: one slot per resident CTA
  double* ws = nullptr;
  std::int64_t slot_doubles = 0;
  int cap_ws = 0;     // rank capacity of a slot
  int ms = 0, ns = 0; // column strides of U (m) and V (n) in a slot
  std::int32_t* rank_out = nullptr;
  // factor write-back (stream levels, write pass), tile-major (planner.h)
  double* W = nullptr;
  const std::int64_t* wx = nullptr;  // W offset of node X's pool
  const std::int32_t* cx = nullptr;  // first column of the pair's segment in X's layout
  const std::int32_t* rx = nullptr;  // column tiles of X's pool
  const std::int64_t* wy = nullptr;
  const std::int32_t* cy = nullptr;
  const std::int32_t* ry = nullptr;
  int row_major = 0;  // pair pools: U / V row-major with row stride rx / ry
  // pivot + packed-LU write-back (proxy levels, write pass): row pivots at
  // piv[piv_off[p] + a], column pivots at piv[piv_off[p] + r + a]
  std::int32_t* piv = nullptr;
  double* lu = nullptr;
  const std::int64_t* piv_off = nullptr;
  const std::int64_t* lu_off = nullptr;
  unsigned* flags = nullptr;
  unsigned long long* counter = nullptr;
  // claim order (claim c -> pair order[c]; nullptr = identity): the costly
  // touching pairs first, so their long ACAs do not form the level's tail
  const std::int32_t* order = nullptr;
  // rank pass, single-pass build: every compressed pair also leaves the
  // reference's own representation (packed LU, r^2 doubles, then its 2r
  // int32 pivots packed into r doubles) in a bump-allocated pool; pool_off[p]
  // = its offset (-1: pool full, kFlagPoolFull raised; -2: rank 0)
  double* pool = nullptr;
  unsigned long long* pool_ctr = nullptr;
  std::int64_t pool_cap = 0;
  std::int64_t* pool_off = nullptr;
};
// threads in {32, 128, 256, 512}; grid = number of workspace slots
void launch_aca(const AcaArgs& a, int threads, int grid, cudaStream_t s);
std::size_t aca_smem_bytes(int threads, int cap_ws);
int aca_blocks_per_sm(int threads, int kernel, std::size_t smem);
// cluster tier (one pair per cluster of `cluster` CTAs, DSMEM reductions)
int aca_max_clusters(int threads, int kernel, int cluster, std::size_t smem);
void launch_aca_cluster(const AcaArgs& a, int threads, int cluster, int nclusters, cudaStream_t s);
// rank-pass pool -> pivots at piv + piv_off[p] (2r int32) and packed LU at
// lu + lu_off[p] (r^2 doubles), one CTA per pair
void launch_aca_compact(const double* pool, const std::int64_t* pool_off, const std::int32_t* rank,
                        std::int64_t npairs, std::int32_t* piv, const std::int64_t* piv_off, double* lu,
                        const std::int64_t* lu_off, cudaStream_t s);
// Explicit factors from the pivots and the triangular inverses of the packed
// LU (lu_invert layout: row-major at inv + inv_off[p], column-major at
// inv + inv_total + inv_off[p]): U = K(X, tau) R^-1 (m x r) and
// V = K(Y, sigma) L^-T (n x r), U V^T = K(X, tau) (L R)^-1 K(sigma, Y), the
// reference's cross approximation (lowrank.cpp:291-327). Written like the
// ACA write pass (tile-major node pools, or row-major pair pools).
struct FactorGenArgs {
  std::int64_t npairs = 0;
  const std::int64_t* xb = nullptr;
  const std::int32_t* m = nullptr;
  const std::int64_t* yb = nullptr;
  const std::int32_t* n = nullptr;
  const std::int32_t* rank = nullptr;
  const std::int32_t* piv = nullptr;      // row pivots (local in X) then col pivots (local in Y)
  const std::int64_t* piv_off = nullptr;
  const double* inv = nullptr;
  std::int64_t inv_total = 0;
  const std::int64_t* inv_off = nullptr;
  const double *px = nullptr, *py = nullptr, *pz = nullptr;
  int kernel = 0;
  double* W = nullptr;
  const std::int64_t* wx = nullptr;
  const std::int32_t* cx = nullptr;
  const std::int32_t* rx = nullptr;
  const std::int64_t* wy = nullptr;
  const std::int32_t* cy = nullptr;
  const std::int32_t* ry = nullptr;
  int row_major = 0;
  int full = 0;  // half levels: X side only, U' = K(X, tau) R^-1 L^-1
  int max_r = 0;
  int rc = 32;  // rows per staged chunk (set by the launcher)
};
void launch_factor_gen(const FactorGenArgs& a, cudaStream_t s);

// -------------------------------------------------------------- matvec.cu
// xp[p] = x[perm[p]], and the weight lane of the packed points p4 (x, y, z, w)
void launch_gather(const double* x, const std::int32_t* perm, std::int64_t n, double* xp, double* p4,
                   cudaStream_t s);
void launch_pack_w(const double* xp, std::int64_t n, double* p4, cudaStream_t s);
void launch_pack_points(const double* px, const double* py, const double* pz, std::int64_t n,
                        double* p4, cudaStream_t s);

struct NodeTable {
  const std::int64_t* rowbeg = nullptr;  // first permuted row of global node g
  const std::int32_t* rows = nullptr;    // number of points
  const std::int64_t* woff = nullptr;    // factor matrix W_g (rows x rpad, row-major)
  const std::int32_t* rpad = nullptr;    // columns of the node's layout
  const std::int64_t* soff = nullptr;    // S_g / proxy slots (rpad entries)
};

struct P1Args {
  const P1Item* items = nullptr;  // one kind per launch
  const StreamDesc* descs = nullptr;  // stream kind: per-item descriptors
  std::int64_t nitems = 0;
  NodeTable nt;
  const double* W = nullptr;
  const double* xp = nullptr;
  const std::int32_t* spos = nullptr;
  double* S = nullptr;
  double* P = nullptr;
  const double *px = nullptr, *py = nullptr, *pz = nullptr;  // permuted points
  const double* p4 = nullptr;  // packed permuted points (x, y, z, x-value)
  const double* q4 = nullptr;  // proxy points (x, y, z, -) in S index space
  const double* q4c = nullptr;  // proxy records centred on their node's box (x', y', z', |.|^2)
  const double* cen = nullptr;  // box centre per global node (4 doubles)
  const std::int32_t* vcols = nullptr;  // per node: leading vertex-partner columns
  unsigned* counter = nullptr;  // dynamic work counter (zeroed before the launch)
};
// persistent CTAs: grid = SMs x per_sm (capped by occupancy and work)
void launch_p1_stream(const P1Args& a, int sms, int per_sm, cudaStream_t s);
void launch_p1_proxy(const P1Args& a, int kernel, int sms, int per_sm, cudaStream_t s);
void launch_phase1_reduce(const P1Reduce* red, std::int64_t nred, NodeTable nt,
                          const std::int32_t* spos, const double* P, double* S,
                          cudaStream_t s);
// q4[i] = (far, far, far, 0) (centred: (far, far, far, 3 far^2)) for i < n
// (padding records, build)
void launch_fill_far(double* q4, std::int64_t n, bool centred, cudaStream_t s);
// q4[so + a] = (x, y, z, .) of the proxy points of every segment (build)
// (and q4c[so + a] = (x - c, y - c, z - c, |.|^2) centred on the segment node's box)
void launch_proxy_gather(const ProxySeg* segs, std::int64_t nseg, const std::int32_t* piv,
                         const double* px, const double* py, const double* pz, const double* cen,
                         double* q4, double* q4c, cudaStream_t s);
// lu holds 2 x lu_total doubles: the packed inverses row-major, then column-major
// in place on S: v (phase-1 output) -> the solved t-vector; persistent CTAs
// (per_sm per SM at most), segments round-robin over the warps (host-sorted
// by decreasing rank), r <= 320
void launch_proxy_solve(const ProxySeg* segs, std::int64_t nseg, const double* lu, std::int64_t lu_total,
                        double* S, int sms, int per_sm, unsigned* counter, cudaStream_t s);
// build time: replace every pair's packed LU by its triangular inverses
// (strict lower L^-1, upper R^-1), row-major at lu and column-major at lu + lu_total
void launch_lu_invert(const ProxySeg* segs, std::int64_t nseg, double* lu, std::int64_t lu_total,
                      int max_r, cudaStream_t s);

struct Phase2Args {
  int depth = 0;
  std::int64_t nleaves = 0;  // leaves processed by this launch
  std::int64_t leaf0 = 0;    // first leaf (Morton id) of this launch
  const std::int64_t* leaf_off = nullptr;  // 8^L + 1
  NodeTable nt;
  const double* W = nullptr;
  const double* S = nullptr;
  const double* xp = nullptr;
  const double *px = nullptr, *py = nullptr, *pz = nullptr;
  const double* p4 = nullptr;  // packed permuted points (x, y, z, x-value)
  const double* q4 = nullptr;  // proxy points (x, y, z, -) in S index space
  const double* q4c = nullptr;  // centred proxy records (x', y', z', |.|^2)
  const double* cen = nullptr;  // box centre per global node (4 doubles)
  const std::int32_t* vcols = nullptr;  // per node: leading vertex-partner columns
  const std::int32_t* perm = nullptr;
  // leaf near lists: self + near_edge + near_face (+ direct partners), CSR
  const std::int32_t* near_off = nullptr;
  const std::int32_t* near_ids = nullptr;
  const std::int32_t* near_dense = nullptr;  // per leaf: leading dense entries (self/edge/face)
  // matrix-free symmetric lists (planner.h): per leaf [self | dense one-way |
  // direct one-way | dense sym | direct sym], category counts, pair-buffer runs
  const std::int32_t* sym_off = nullptr;
  const std::int32_t* sym_ids = nullptr;
  const std::int32_t* sym_cnt = nullptr;
  const std::int64_t* out_off = nullptr;
  double* pairbuf = nullptr;
  // stored near field (near_mode 0): per owned leaf a row-major
  // m x nf_cols block of its dense sources in symmetric-list order (planner.h)
  const std::int64_t* nf_off = nullptr;
  const std::int32_t* nf_cols = nullptr;
  const double* NF = nullptr;
  int nf_mask = 0;  // planner.h set_near_storage: bit 0 dense, bit 1 direct sources stored
  int kernel = 0;
  double diag = 0.0;
  double* b = nullptr;          // output, original order
  double* cpart_out = nullptr;  // near/direct partial sums (Morton order) when levels add partials
  std::int64_t lbase[24] = {0};  // node_base per level (by value)
  int mode[24] = {0};            // LevelMode per level
  unsigned* counter = nullptr;   // p2_compute work counter (zeroed before the launch)
  unsigned* counter2 = nullptr;  // p2_stream work counter
  // node-major proxy pass (thread = target row): when set, p2_compute skips
  // the proxy ranges and p2_proxy writes one partial per proxy level
  const P2Item* p2_items = nullptr;
  std::int64_t n_p2_items = 0;
  // half levels, regenerated side: both uses per entry (planner.h H2Item)
  const H2Item* h2_items = nullptr;
  std::int64_t n_h2_items = 0;
  unsigned* counter_h2 = nullptr;
  const std::int32_t* spos = nullptr;
  double* Sw = nullptr;  // S, written by the half-level pass (its v)
  double* P = nullptr;   // v partials of multi-chunk nodes
  // stream levels: one row tile per item, one partial per stream level
  const P2Item* p2s_items = nullptr;
  const StreamDesc* p2s_descs = nullptr;
  std::int64_t n_p2s_items = 0;
  double* lvl_part = nullptr;  // [levels with phase-2 work x N] (Morton order)
  // p2_stream: its producer holds the first copy until *wait_flag reaches
  // wait_value (set on the FP64 lane after the solves), so the HBM lane's
  // CTAs can be resident early without competing with the solves. A bounded
  // throttle, not a dependency: it gives up after kFlagWaitLimitNs
  const unsigned* wait_flag = nullptr;
  unsigned wait_value = 0;
  std::int64_t n_total = 0;    // N
  unsigned* counter3 = nullptr;
};
// matrix-free near field + direct leaf blocks (near_mode on-the-fly); near
// lists of at most kMaxNearRanges leaves (HODLR3D: 27 dense + <= 189 direct)
constexpr int kMaxNearRanges = 256;
// matrix-free near field + direct leaf blocks (near_mode on-the-fly)
void launch_p2_near(const Phase2Args& a, int sms, int per_sm, cudaStream_t s);
void launch_p2_stream(const Phase2Args& a, int sms, int per_sm, cudaStream_t s);
void launch_half2(const Phase2Args& a, int sms, int per_sm, cudaStream_t s);
void launch_p2_proxy(const Phase2Args& a, int sms, int per_sm, cudaStream_t s);
// *flag = value (release, device scope), stream-ordered
void launch_set_flag(unsigned* flag, unsigned value, cudaStream_t s);
// b[perm[p]] = cpart[p] + incoming pair-buffer runs of p's leaf (ascending
// partner, may be null) + sum over levels (in order) of lvl_part[l][p];
// one warp per owned leaf
void launch_combine(const double* cpart, const double* lvl_part, int n_lvl, std::int64_t n_total,
                    const std::int64_t* leaf_off, std::int64_t leaf0, std::int64_t nleaves,
                    const std::int32_t* in_off, const std::int64_t* in_pos, const double* pairbuf,
                    const std::int32_t* perm, double* b, double* bm, cudaStream_t s);
// after the all-gather of the Morton-order b: the rows other shards own
void launch_unpermute_rest(const double* bm, const std::int32_t* perm, std::int64_t n, std::int64_t row0,
                           std::int64_t row1, double* b, cudaStream_t s);

// ---------------------------------------------------------------- pair.cu
constexpr int kPairMaxRp = 128;  // pair levels: ranks above this stay two-phase
struct PairArgs {
  const PairDesc* descs = nullptr;
  std::int64_t n = 0;
  const double* W = nullptr;
  const double* xp = nullptr;
  double* out = nullptr;
};
std::size_t pair_smem_bytes();
// persistent, per_sm CTAs per SM; pairs interleaved statically over the CTAs
void launch_pair(const PairArgs& a, int sms, int per_sm, cudaStream_t s);
void launch_pair_gather(const P2Item* items, std::int64_t nitems, const std::int64_t* rowbeg,
                        const std::int32_t* pc_off, const std::int64_t* pc_pos, const double* out,
                        double* lvl, std::int64_t n_total, cudaStream_t s);

// --------------------------------------------------------------- fused.cu
constexpr int kFusedMaxRank = 128;  // fused levels: ranks above this stay two-phase
struct FusedArgs {
  const FusedDesc* descs = nullptr;
  std::int64_t n = 0;
  const double* p4 = nullptr;  // permuted (x, y, z, x-value)
  const std::int32_t* piv = nullptr;
  const double* lu = nullptr;  // triangular inverses (lu_invert_kernel)
  std::int64_t lu_total = 0;
  double* out = nullptr;       // pair-output buffer
  unsigned long long* prof = nullptr;  // optional: per-CTA phase cycle sums (kFusedProfSlots each)
};
constexpr int kFusedProfSlots = 6;  // setup, evaluation, v exchange, solve, apply, pairs
int fused_max_node();  // points per node of a fused pair
void launch_fused(const FusedArgs& a, int kernel, int sms, cudaStream_t s);

// --------------------------------------------------------------- gmres.cu
std::size_t dot_scratch_doubles();
// *out = a . b (or its square root), fixed-order two-stage reduction
void launch_dot(const double* a, const double* b, std::int64_t n, double* scratch, double* out, bool sqrt_of,
                cudaStream_t s);
// y += c x with c = sign * (*cdev) if cdev else chost
void launch_axpy(double* y, const double* x, std::int64_t n, const double* cdev, double sign, double chost,
                 cudaStream_t s);
void launch_scale_div(double* y, const double* x, std::int64_t n, const double* d, cudaStream_t s);
void launch_affine(double* w, const double* v, std::int64_t n, double alpha, double beta, cudaStream_t s);
void launch_sub(double* r, const double* f, const double* w, std::int64_t n, cudaStream_t s);
// exact dense product (diagonal rule) from the packed Morton-order points,
// b in original order
void launch_direct(const double* p4, std::int64_t n, int kernel, double diag, const std::int32_t* perm,
                   double* b, cudaStream_t s);
// exact row sums (K x)[p] at Morton positions rows[0..nrows) (reference_error)
void launch_exact_rows(const double* p4, std::int64_t n, int kernel, double diag, const std::int64_t* rows,
                       std::int64_t nrows, double* out, unsigned* flags, cudaStream_t s);

// ------------------------------------------------------------------ ie.cpp
double unit_cell_integral_constant();
double cell_self_integral(double h);
void tensor_grid_points(std::int64_t n, double* xyz);

// Build-time near-field scan: coincidence check (and optional store).
void launch_near_scan(const Phase2Args& a, double* NF_out, unsigned* flags, cudaStream_t s);

}  // namespace h3db
