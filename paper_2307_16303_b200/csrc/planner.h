// Host-side planning of the HODLR3D representation and of the matvec launch
// plan (pure C++, no CUDA): which pairs a shard compresses, the node-major
// column layout shared by the factor pool W, the t-vector pool S and the
// proxy lists, the phase-1 work items, the triangular-solve segments and the
// leaf near lists. Exposed through the C-ABI (h3d_plan_*) so the multi-GPU
// shard logic is testable on CPU (tests/test_shard_plan.py, gloo world 2).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace h3db {

// Stream-level factor pools are tile-major: W_Z (rows x rpad, rows padded to
// kTileRows, rpad to kTileCols) is stored as kTileRows x kTileCols row-major
// tiles, tile (rt, ct) at woff + (rt * rpad / kTileCols + ct) * kTileDoubles,
// so every tile is one contiguous 8 KB bulk copy (cp.async.bulk) for both the
// column sums of phase 1 and the row dots of phase 2.
// rows per pass of the matrix-free near kernel (7 consumer warps x 7 rows);
// only leaves within one pass take part in the symmetric pair evaluation
constexpr int kNearPassRows = 49;
constexpr int kTileRows = 16;
constexpr int kTileCols = 64;
constexpr int kTileDoubles = kTileRows * kTileCols;
#ifdef __CUDACC__
#define H3D_HD __host__ __device__
#else
#define H3D_HD
#endif
H3D_HD inline std::int64_t tile_index(std::int64_t i, std::int64_t c, std::int64_t nct) {
  return ((i / kTileRows) * nct + c / kTileCols) * kTileDoubles + (i % kTileRows) * kTileCols +
         c % kTileCols;
}

// How the admissible blocks of one level are applied in the matvec.
enum LevelMode : int {
  kModeStream = 0,  // explicit ACA factors streamed from the pool W (2 x 8 r(m+n) B)
  kModeProxy = 1,   // matrix-free: pivots + packed LU (reference lowrank.cpp:291-327),
                    //   2 r(m+n) kernel evaluations + 2 r^2 solve FMAs per pair
  kModeDirect = 2,  // exact dense evaluation (leaf level only): 2 m n evaluations per pair
  kModePair = 3,    // explicit factors, pair-major: one fused pass per pair reads U and V
                    //   once (8 r(m+n) B), both products through a per-pair output buffer
  kModeFused = 4,   // matrix-free like kModeProxy, pair-major: r(m+n) kernel evaluations per
                    //   pair, each entry kept in shared memory for both orientations
  kModeHalf = 5,    // half explicit, half regenerated, no solves: U' = K(X, tau) (LR)^-1
                    //   (m x r) streamed, K(sigma, Y) regenerated; 2 x 8 r m B + 2 r n
                    //   evaluations per pair. Every node carries two column groups: the
                    //   pairs it is X of (stream kernels, its own node id) and the pairs
                    //   it is Y of (proxy kernels, a virtual node id >= total_nodes())
  kModeSplit = 6,   // matrix-free like kModeProxy, three passes: the pairs a node is X of
                    //   (proxy kernels, node id gid) evaluated in phase 1 and phase 2, the
                    //   pairs it is Y of (virtual node id gv) once, both uses in the two-use
                    //   pass between two solve rounds: 1.5 r(m+n) evaluations per pair
};
constexpr int kModeLast = kModeSplit;
// levels whose nodes carry two column groups (gid: the pairs a node is X of,
// gv: the pairs it is Y of)
inline bool two_groups(int mode) { return mode == kModeHalf || mode == kModeSplit; }

// Fused proxy pass (kModeFused levels, fused.cu): pivots sigma (row, in X) at
// piv_off, tau (column, in Y) at piv_off + r; inverses at lu_off (row-major)
// and lu_off + lu_total (column-major); outputs like PairDesc.
struct FusedDesc {
  std::int64_t piv_off, lu_off;
  std::int64_t xrow, yrow;
  std::int64_t out;
  std::int32_t m, n, r, own;
  std::int32_t touch;  // 1: the boxes touch (difference form of r^2)
  std::int32_t pad;
  double cx, cy, cz;   // pair centre (midpoint of the two box centres)
  double pad2;
};

// Fused pair pass (kModePair levels): F = [U; V] ((m + n) x rp, row-major,
// rp = r rounded up to even) at woff; t_U = U^T x_X, t_V = V^T x_Y; outputs
// U t_V (m rows, for X) and V t_U (n rows, for Y) at out.
struct PairDesc {
  std::int64_t woff;
  std::int64_t xrow, yrow;  // first permuted row of X and of Y
  std::int64_t out;         // pair-output buffer offset (X's rows, then Y's)
  std::int32_t m, n, rp, own;  // own: bit 0 = X owned here, bit 1 = Y owned
};

// Two boxes of one level touch (Chebyshev distance 1 between their Morton
// ids' grid coordinates)
bool boxes_touch(std::int64_t a, std::int64_t b);

// Variants, h3d::Variant order (reference octree.hpp:80)
constexpr int kVariantHodlr3d = 0;
constexpr int kVariantHodlr = 1;
constexpr int kVariantHStrong = 2;
constexpr int kListKinds = 4;

struct LevelLists {
  // CSR per kind: 0 inter, 1 near_edge, 2 near_face, 3 near_vertex (reference
  // NodeLists, octree.hpp:88-93; near_vertex only for H-strong). Kinds 1..3
  // are the dense leaf blocks (hmatrix.cpp:105-120).
  std::vector<std::int32_t> off[kListKinds];
  std::vector<std::int32_t> ids[kListKinds];
};

struct LevelPairs {
  std::vector<std::int32_t> X, Y;  // Morton ids, X < Y
  std::vector<std::int32_t> rank;
  std::vector<std::int32_t> eX, eY;  // inter-list entry of Y in X's list / X in Y's list
  int threads = 32;                  // ACA CTA size (fixed per level: determinism)
  int cluster = 0;                   // ACA CTAs per pair (0 = not chosen yet)
  int max_m = 0, max_n = 0, max_mn = 0;
};

// phase-1 work item (both stream and proxy kinds)
struct P1Item {
  std::int32_t node;   // global node id
  std::int32_t row0;   // stream: first row; proxy: first source point (local)
  std::int32_t nrows;
  std::int32_t col0;   // first column (local to the node's column layout)
  std::int32_t ncols;  // <= 256
  std::int32_t kind;   // kModeStream / kModeProxy
  std::int64_t pslot;  // -1: write to S through spos; else partial buffer base
};

// phase-2 item: targets = rows [row0, row0 + nrows) of node `node`; proxy
// levels: <= 256 rows, sources = the node's proxy list; stream levels: one
// row tile (<= kTileRows rows) dotted with S_node. slot = output partial
// (one per level with phase-2 work, summed in level order by combine)
struct P2Item {
  std::int32_t node;
  std::int32_t row0;
  std::int32_t nrows;
  std::int32_t slot;
};

// Half levels (kModeHalf), the regenerated side: one pass per row chunk of a
// node's virtual group evaluates every entry E = K(sigma, rows) once for
// both of its uses - b rows += E^T t (t = the partners' streamed U'^T x,
// ready once p1_stream is done) and v = E x_rows (the partners' streamed
// phase-2 weights, scattered through spos, or partials at pslot when the
// node spans several chunks, summed by a P1Reduce of kind kModeHalf).
struct H2Item {
  std::int32_t node;   // virtual node id (planner: gv)
  std::int32_t row0;
  std::int32_t nrows;  // <= 256
  std::int32_t slot;   // output partial of the rows
  std::int64_t pslot;  // -1: v through spos; else this chunk's partial base
};

// Device descriptor of one stream-level work item (engine.cu, from P1Item /
// P2Item + the node tables), so the bulk-copy producer needs one load per item.
struct StreamDesc {
  std::int64_t wbase;  // W offset of the item's first tile
  std::int64_t aux;    // phase 1: first x row (permuted); phase 2: slot * N + first row
  std::int64_t sbase;  // phase 2: S offset of the node's columns
  std::int32_t nrt;    // row tiles
  std::int32_t ncti;   // column tiles in the item
  std::int32_t nct;    // column tiles of the node (tile-row stride)
  std::int32_t nrows;  // rows
  std::int32_t ncols;  // phase 1: columns
  std::int32_t pad;
};

struct P1Reduce {
  std::int32_t node;
  std::int32_t ncols;
  std::int32_t nchunks;
  std::int32_t kind;   // LevelMode of the node's level (the two kinds reduce on different streams)
  std::int64_t pbase;  // partials: pbase + chunk * ncols + c
};

// One ordered proxy block (target Z, partner k): its S segment, pivots, LU.
struct ProxySeg {
  std::int64_t so;       // S-space offset of the segment (soff[Z] + column offset)
  std::int64_t base;     // first permuted point index of the partner node k
  std::int64_t piv_off;  // offset of the pair's pivots (row pivots at piv_off, col at piv_off + r... see engine)
  std::int64_t lu_off;   // offset of the pair's packed LU (row-major r x r)
  std::int32_t r;
  std::int32_t side;     // 0: Z is the pair's row side X (proxies = col pivots tau in k)
                         // 1: Z is the pair's col side Y (proxies = row pivots sigma in k)
  std::int32_t solve;    // 1 if Z is owned here (its S segment is solved before phase 2)
  std::int32_t node;     // global node id of Z
};

struct PlanSizes {
  std::int64_t w_doubles = 0, s_doubles = 0, p_doubles = 0, piv_total = 0, lu_total = 0;
  std::int64_t factor_doubles = 0, proxy_units = 0, half_units = 0, direct_evals = 0, sum_rank = 0,
               npairs = 0, nblocks_ordered = 0;
  std::int64_t near_blocks = 0, near_entries = 0;
  int max_rank = 0;
  std::uint64_t ref_float_count = 0, ref_int_count = 0;
};

class Planner {
 public:
  Planner(int depth, std::int64_t n, std::vector<std::vector<std::int64_t>> off,
          std::vector<LevelLists> lists, int rank, int world, std::vector<int> modes);

  int depth() const { return L_; }
  int mode(int l) const { return mode_[l]; }
  const std::vector<int>& modes() const { return mode_; }
  // stream <-> proxy may change after the rank pass (direct cannot: it decides
  // which pairs exist)
  // the rank-independent part of layout() (leaf plan, near-field lists);
  // layout() runs it when it has not run yet
  void layout_leaf();
  // stored near field (nf_*): bit 0 = the dense leaf blocks (self, edge,
  // face: the reference's DenseMode::Cached), bit 1 = the direct leaf-level
  // admissible blocks; set before layout_leaf()
  void set_near_storage(int mask) { nf_mask_ = mask; }
  int near_storage() const { return nf_mask_; }
  void set_mode(int l, int m) {
    if (mode_[l] == kModeDirect || m == kModeDirect)
      throw std::invalid_argument("planner: direct mode is fixed at construction");
    if (m < 0 || m > kModeLast) throw std::invalid_argument("planner: bad level mode");
    mode_[l] = m;
  }
  bool owned(int level, std::int64_t m) const;
  std::int64_t gid(int level, std::int64_t m) const { return node_base_[level] + m; }
  std::int64_t node_size(int level, std::int64_t m) const {
    return off_[level][m + 1] - off_[level][m];
  }
  std::int64_t total_nodes() const { return node_base_.back(); }
  // half levels: node z's regenerated column group has node id vbase[l] + z
  // (after every real node); -1 elsewhere. Valid after layout().
  std::vector<std::int64_t> vbase;
  std::int64_t gv(int level, std::int64_t m) const { return vbase[level] + m; }
  const std::vector<std::int64_t>& node_base() const { return node_base_; }
  const std::vector<std::vector<std::int64_t>>& offsets() const { return off_; }
  const std::vector<LevelLists>& lists() const { return lists_; }

  LevelPairs& pairs(int l) { return pairs_[l]; }
  const LevelPairs& pairs(int l) const { return pairs_[l]; }

  // After every level's ranks are set: column layout, S, spos, per-pair write
  // offsets, proxy segments, phase-1 items, leaf plan.
  void layout();

  // results ----------------------------------------------------------------
  std::vector<std::int64_t> woff, soff, rowbeg;
  std::vector<std::int32_t> rpad, rows;
  // columns of vertex-adjacent partners come first in every node's layout:
  // vcols[g] of them. Entries against those partners can be arbitrarily
  // close; the rest are at least one box apart (the regenerating kernels
  // use a cancellation-prone r^2 form only there)
  std::vector<std::int32_t> vcols;
  // phase-1 column ranges per node: [0, p1a) and [p1b, p1c) (columns whose
  // partner's t-vector is consumed on this shard; all columns on one shard)
  std::vector<std::int32_t> p1a, p1b, p1c;
  std::vector<double> center;  // 4 per global node: box centre (x, y, z, 0)
  std::vector<std::int32_t> spos;
  // per level, per pair: stream levels: W node base (pair_wx/wy), first column
  // of the pair's segment (pair_cx/cy) and column tiles of the node
  // (pair_rx/ry = rpad / kTileCols); proxy levels: pivot/LU offsets
  std::vector<std::vector<std::int64_t>> pair_wx, pair_wy, pair_piv, pair_lu;
  std::vector<std::vector<std::int32_t>> pair_rx, pair_ry, pair_cx, pair_cy;
  std::vector<ProxySeg> proxy_segs;
  std::vector<P1Item> items;
  std::vector<P1Reduce> reds;
  std::vector<P2Item> p2_items;   // owned nodes of proxy levels, <= 256 rows each
  std::vector<P2Item> p2s_items;  // owned nodes of stream levels, one row tile each
  std::vector<H2Item> h2_items;   // half levels: the regenerated side, both uses in one pass
  // pair levels: one descriptor per pair with an owned side (grouped by level),
  // pd_level[l] .. pd_level[l + 1]; per owned node the output runs of its
  // pairs (pc_off over global nodes, pc_pos in pair order), gathered into the
  // level's partial by pg_items (owned nodes, <= 256 rows each)
  std::vector<PairDesc> pair_descs;
  std::vector<std::int64_t> pd_level;
  // fused levels: one descriptor per pair with an owned side (grouped by
  // level, fd_level[l] .. fd_level[l + 1]); outputs share pair_out / pc_* /
  // pg_items; pg_level[l] .. pg_level[l + 1] = the level's gather items
  std::vector<FusedDesc> fused_descs;
  std::vector<std::int64_t> fd_level, pg_level;
  std::vector<std::int32_t> pc_off;
  std::vector<std::int64_t> pc_pos;
  std::vector<P2Item> pg_items;
  std::int64_t pair_out_total = 0;
  int n_proxy_levels = 0;         // output slots of the phase-2 proxy + stream passes
  std::int64_t leaf0 = 0, leaf1 = 0;
  std::vector<std::int32_t> near_off, near_ids;
  std::vector<std::int32_t> near_dense;  // per leaf: leading dense entries (self, edge, face)
  // matrix-free near field with the symmetry used once per owned pair: per
  // owned leaf X the list [self | dense one-way | direct one-way | dense sym |
  // direct sym] (sym_cnt: the four counts); "sym" = owned partner Y > X, its
  // entries evaluated once for X's rows and (column sums) Y's rows, Y's part
  // written to the pair buffer at out_off[X] + (flattened index - sym start);
  // partners Y < X owned are omitted (their pass supplies X's part, in_off /
  // in_pos = X's incoming pair-buffer runs, ascending Y); "one-way" = Y owned
  // by another shard.
  std::vector<std::int32_t> sym_off, sym_ids, sym_cnt;
  std::vector<std::int64_t> out_off;  // nl + 1
  std::vector<std::int32_t> in_off;   // nl + 1
  std::vector<std::int64_t> in_pos;
  // stored near field: per owned leaf X a row-major m x nf_cols[X] block at
  // nf_off[X], one column per STORED source of X's symmetric list in list
  // order (self, dense one-way, direct one-way, dense sym, direct sym; dense
  // ones with storage bit 0, direct ones with bit 1) - exactly the values the
  // matrix-free near pass evaluates, in its order (bitwise-equal results)
  std::vector<std::int64_t> nf_off;
  std::vector<std::int32_t> nf_cols;
  std::int64_t nf_total = 0;
  std::int64_t row0 = 0, row1 = 0;  // owned permuted rows
  std::vector<std::int64_t> rank_row0, rank_row1;
  PlanSizes sizes;

 private:
  void build_pairs();

  int L_;
  bool leaf_done_ = false;
  int nf_mask_ = 1;
  std::int64_t n_;
  std::vector<std::vector<std::int64_t>> off_;
  std::vector<LevelLists> lists_;
  int rank_, world_, oct0_, oct1_;
  std::vector<int> mode_;
  std::vector<std::int64_t> node_base_;
  std::vector<LevelPairs> pairs_;
  std::vector<std::vector<std::int32_t>> entry_pair_, entry_col_;
};

// Cost-model default for the per-level modes: the leaf level
// is evaluated directly when its blocks are smaller than their factors.
std::vector<int> default_modes(int depth, std::int64_t n, int policy);

}  // namespace h3db
